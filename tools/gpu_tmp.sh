mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_band_wcol --launch-skip 4 --launch-count 2 -f -o gpurun_out/r02e_wcol_cfg4 python tools/probe_strips.py 512 4096 > gpurun_out/ncu_wcol.log 2>&1
PINTGPU_GRAPHS=0 timeout 1200 python tools/probe_breakdown.py cfg4 merge > gpurun_out/bd_cfg4_strips_ch1024.txt 2>&1
