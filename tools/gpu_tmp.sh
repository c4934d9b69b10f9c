mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/ab_tests.log 2>&1
timeout 600 python tools/probe_scaling.py > gpurun_out/scal.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/ab.csv python tools/probe_scaling.py 512 > /dev/null 2>&1
python tools/ncu_sum.py gpurun_out/ab.csv 14 >> gpurun_out/scal.log
