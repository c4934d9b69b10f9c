mkdir -p gpurun_out; ./tools/mb/rhs_mb_8 > gpurun_out/mb8.log 2>&1; ./tools/mb/rhs_mb_16 > gpurun_out/mb16.log 2>&1
