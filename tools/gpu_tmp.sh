mkdir -p gpurun_out
rm -f /tmp/strips_*.npy
for B in 256 4096; do
( PG_STRIPS=0 timeout 900 python tools/probe_strips.py 512 $B; PG_STRIPS=1 timeout 900 python tools/probe_strips.py 512 $B ) > gpurun_out/strips_rhs_512_B$B.txt 2>&1
rm -f /tmp/strips_*.npy
done
( PG_STRIPS=0 timeout 900 python tools/probe_strips.py 256 4096; PG_STRIPS=1 timeout 900 python tools/probe_strips.py 256 4096 ) > gpurun_out/strips_rhs_256.txt 2>&1
