# factor slab allocation check + rhs ncu capture
mkdir -p gpurun_out
L=gpurun_out/setup_ab.log
: > $L
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py tests/test_gpu_edge.py -x -q > gpurun_out/setup_tests.log 2>&1; tail -2 gpurun_out/setup_tests.log >> $L
echo "== e2e setup split (slab)" >> $L
PG_DEBUG_SETUP=1 timeout 600 python bench.py --no-cpu --no-phi --no-seq > gpurun_out/bench_dbg.json 2>> $L
python -c "import json;d=json.load(open('gpurun_out/bench_dbg.json'));print(d['value'], d['e2e'])" >> $L
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_band_rhs_dia --launch-skip 3 -c 1 -o gpurun_out/rhs_full python tools/probe_band.py cfg2 0:1024 > gpurun_out/ncu_rhs.log 2>&1
