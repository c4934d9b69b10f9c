# rhs A/B (k_band_rhs_dia vs cp.async ring)
mkdir -p gpurun_out
L=gpurun_out/rhs_ab.log
: > $L
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/rhs_tests.log 2>&1; tail -2 gpurun_out/rhs_tests.log >> $L
for v in 0 2; do
  echo "== PG_RHS_SM=$v" >> $L
  PG_RHS_SM=$v timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:rhs --csv --log-file gpurun_out/rhs_ab$v.csv python tools/probe_band.py cfg2 0:1024 0:64 > /dev/null 2>&1
  python tools/ncu_sum.py gpurun_out/rhs_ab$v.csv 6 >> $L
done
PG_RHS_SM=2 timeout 300 python tools/probe_breakdown.py cfg2 >> $L 2>&1
PG_RHS_SM=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_band_rhs_cp --launch-skip 3 -c 1 -o gpurun_out/rhs_cp2_full python tools/probe_band.py cfg2 0:1024 > gpurun_out/ncu_rhs.log 2>&1
