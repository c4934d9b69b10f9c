# per-(grid, batch) Phi breakdown of one config-4 (and config-2) solve
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/bd_clocks.txt
timeout 600 python tools/probe_breakdown.py cfg4 merge > gpurun_out/bd_cfg4.txt 2>&1
timeout 300 python tools/probe_breakdown.py cfg2 > gpurun_out/bd_cfg2.txt 2>&1
