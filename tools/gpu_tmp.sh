mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_ring -c 1 -o gpurun_out/factor python tools/probe_band.py cfg2 0:64 > gpurun_out/ncu_factor.log 2>&1
