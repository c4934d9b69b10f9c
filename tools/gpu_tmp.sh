mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strips.py -q --durations=5 > gpurun_out/pytest_strips.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strips.log
