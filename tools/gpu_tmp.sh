mkdir -p gpurun_out
PINTGPU_GRAPHS=0 timeout 1200 python tools/probe_breakdown.py cfg4 merge > gpurun_out/bd_cfg4_strips4.txt 2>&1
