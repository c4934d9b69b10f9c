mkdir -p gpurun_out
PG_DEBUG_SETUP=1 timeout 600 python tools/probe_band.py cfg4 1:256 0:1 > gpurun_out/probe_band_fac.txt 2>&1
PG_DEBUG_SETUP=1 timeout 600 python tools/probe_band.py cfg2 0:1024 > gpurun_out/probe_band_fac2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_phi.py -q -k "cholesky or wide" > gpurun_out/pytest_fac.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fac.log
