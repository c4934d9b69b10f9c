mkdir -p gpurun_out
PG_DEBUG_SETUP=1 timeout 900 python tools/probe_e2e4.py > gpurun_out/e2e4.txt 2>&1
