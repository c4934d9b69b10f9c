mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_strips.py -q -x > gpurun_out/pytest_strips.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strips.log
