mkdir -p gpurun_out
PG_DEBUG_SETUP=1 timeout 900 python tools/probe_e2e4.py > gpurun_out/e2e4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_strips.py tests/test_gpu_phi.py tests/test_gpu_mgrit.py tests/test_gpu_edge.py -q > gpurun_out/pytest_strips.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strips.log
