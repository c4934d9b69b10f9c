mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/ab_tests.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:rhs --csv --log-file gpurun_out/ab.csv python tools/probe_band.py cfg2 0:1024 0:64 > /dev/null 2>&1
python tools/ncu_sum.py gpurun_out/ab.csv 6 > gpurun_out/ab.log
timeout 300 python tools/probe_breakdown.py cfg2 >> gpurun_out/ab.log 2>&1
