# rhs A/B (staged k_band_rhs_sm vs k_band_rhs_dia) + e2e setup split
mkdir -p gpurun_out
L=gpurun_out/rhs_ab.log
: > $L
PG_RHS_SM=1 timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/rhs_tests.log 2>&1; tail -2 gpurun_out/rhs_tests.log >> $L
for v in 0 1; do
  echo "== PG_RHS_SM=$v" >> $L
  PG_RHS_SM=$v timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:rhs --csv --log-file gpurun_out/rhs_ab$v.csv python tools/probe_band.py cfg2 0:1024 0:64 > /dev/null 2>&1
  python tools/ncu_sum.py gpurun_out/rhs_ab$v.csv 6 >> $L
  PG_RHS_SM=$v timeout 300 python tools/probe_breakdown.py cfg2 >> $L 2>&1
done
echo "== e2e setup split" >> $L
PG_DEBUG_SETUP=1 timeout 600 python bench.py --no-cpu --no-phi --no-seq > gpurun_out/bench_dbg.json 2>> $L
