# k_band_rb: parity tests, then per-call A/B against the round-1 kernels
mkdir -p gpurun_out
O=gpurun_out/rb_ab.log
: > $O
timeout 600 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -x -q > gpurun_out/rb_tests.log 2>&1
echo "tests rc=$?" >> $O
for cfg in "PG_BAND_RB=0" "PG_BAND_RB=1" "PG_BAND_RB=1 PG_RB_ALT=1" "PG_BAND_RB=1 PG_RB_ALT=2"; do
  echo "== $cfg cfg2" >> $O
  env $cfg timeout 300 python tools/probe_band.py cfg2 0:1024 0:64 >> $O 2>&1
done
for cfg in "PG_BAND_RB=0" "PG_BAND_RB=1" "PG_BAND_RB=1 PG_RB_ALT=1" "PG_BAND_RB=1 PG_BAND_BC=16" "PG_BAND_RB=1 PG_BAND_BC=16 PG_RB_ALT=1"; do
  echo "== $cfg cfg4" >> $O
  env $cfg timeout 300 python tools/probe_band.py cfg4 0:4096 0:1024 1:256 >> $O 2>&1
done
