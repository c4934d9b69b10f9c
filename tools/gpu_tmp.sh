mkdir -p gpurun_out
PG_BAND_BC=16 PG_RB_ALT=1 PG_RB_NBUF=2 timeout 600 python tools/probe_band.py cfg4 0:4096 2>&1 | tail -1 > gpurun_out/probe_bc16_2cta.txt
PG_BAND_BC=16 PG_RB_ALT=1 timeout 600 python tools/probe_band.py cfg4 0:4096 2>&1 | tail -1 > gpurun_out/probe_bc16_alt1.txt
PG_BAND_BC=16 timeout 600 python tools/probe_band.py cfg4 0:4096 2>&1 | tail -1 > gpurun_out/probe_bc16.txt
timeout 600 python -m pytest tests/test_gpu_dropin.py -q > gpurun_out/pytest_dropin.log 2>&1
