mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
timeout 300 python tools/probe_band.py cfg2 > gpurun_out/ab.log 2>&1
timeout 300 python tools/probe_breakdown.py cfg2 >> gpurun_out/ab.log 2>&1
