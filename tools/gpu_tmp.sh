mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/ab_tests.log 2>&1
timeout 600 python tools/probe_scaling.py > gpurun_out/scal.log 2>&1
timeout 300 python tools/probe_breakdown.py cfg2 >> gpurun_out/scal.log 2>&1
