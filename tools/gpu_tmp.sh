mkdir -p gpurun_out
for t in 32 16 8 4; do PG_RHS_CCT=$t timeout 600 python tools/probe_band.py cfg4 0:4096 2>&1 | tail -1 > gpurun_out/probe_rhs_cc$t.txt; done
