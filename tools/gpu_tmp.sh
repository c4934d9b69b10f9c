mkdir -p gpurun_out
for t in 2 3 4 5 6 7; do PG_STRIPS=0 PG_RHS_T=$t timeout 600 python tools/probe_band.py cfg4 0:4096 2>&1 | tail -1 > gpurun_out/probe_rhs_u$t.txt; done
