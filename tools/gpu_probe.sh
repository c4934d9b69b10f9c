mkdir -p gpurun_out
timeout 300 python tools/probe_e2e.py > gpurun_out/probe_e2e.log 2>&1
timeout 300 python tools/probe_breakdown.py cfg2 > gpurun_out/probe_breakdown.log 2>&1
