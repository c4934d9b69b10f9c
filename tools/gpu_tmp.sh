mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_full.py tests/test_gpu_mgrit.py -q > gpurun_out/pytest_fac.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fac.log
PG_DEBUG_SETUP=1 timeout 600 python tools/probe_band.py cfg4 0:4096 1:256 > gpurun_out/probe_band_fac.txt 2>&1
PG_DEBUG_SETUP=1 timeout 600 python tools/probe_band.py cfg2 0:1024 > gpurun_out/probe_band_fac2.txt 2>&1
