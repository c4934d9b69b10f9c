# SPIKE fix A/B against the previous build (per-kernel ncu times + breakdown)
mkdir -p gpurun_out
L=gpurun_out/fix_ab.log
: > $L
timeout 600 python -m pytest tests/test_gpu_mgrit.py -x -q > gpurun_out/fix_tests.log 2>&1; tail -2 gpurun_out/fix_tests.log >> $L
for lib in base new; do
  echo "== $lib" >> $L
  if [ $lib = base ]; then export PINTGPU_LIB=$PWD/paper_1912_03106_b200/lib/libpintgpu_base.so; else unset PINTGPU_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spike_fix --csv --log-file gpurun_out/fix_$lib.csv python tools/probe_breakdown.py cfg2 > /dev/null 2>&1
  python tools/ncu_sum.py gpurun_out/fix_$lib.csv 6 >> $L
  timeout 300 python tools/probe_breakdown.py cfg2 >> $L 2>&1
done
