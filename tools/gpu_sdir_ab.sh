# k_sdir A/B: occupancy (MINB) and columns per CTA; then the full bench line
mkdir -p gpurun_out
L=gpurun_out/sdir_ab.log
: > $L
for v in "PG_SDIR_MINB=3" "PG_SDIR_MINB=4" "PG_DIA_CTA_KB=100" "PG_DIA_CTA_KB=30 PG_SDIR_MINB=4" "PG_DIA_CTA_KB=30"; do
  echo "== $v" >> $L
  env $v timeout 300 python tools/probe_cfg5.py 256 1024 >> $L 2>&1
done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
