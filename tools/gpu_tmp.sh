mkdir -p gpurun_out; ./tools/mb/rhs_mb > gpurun_out/mb.log 2>&1
