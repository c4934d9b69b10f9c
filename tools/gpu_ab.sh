mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/ab_tests.log 2>&1
for v in "PG_BORDER_CL=0" "PG_BORDER_CL=1" "PG_SPIKE_CHUNKS=12" "PG_SPIKE_CHUNKS=16"; do
echo "== $v" >> gpurun_out/ab.log
env $v timeout 300 python tools/probe_breakdown.py cfg2 >> gpurun_out/ab.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:border --csv --log-file gpurun_out/ab.csv python tools/probe_band.py cfg2 0:64 1:64 > /dev/null 2>&1
python tools/ncu_sum.py gpurun_out/ab.csv 6 >> gpurun_out/ab.log
