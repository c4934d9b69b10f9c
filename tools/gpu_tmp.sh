mkdir -p gpurun_out
rm -f /tmp/strips_*.npy
( PG_STRIPS=0 timeout 900 python tools/probe_strips.py 512 4096; PG_STRIPS=1 timeout 900 python tools/probe_strips.py 512 4096 ) > gpurun_out/strips_512.txt 2>&1
