mkdir -p gpurun_out
rm -f /tmp/strips_*.npy
for B in 1 4; do
( PG_STRIPS=0 timeout 900 python tools/probe_strips.py 512 $B; PG_STRIPS_SMALL_MIN=1 timeout 900 python tools/probe_strips.py 512 $B ) > gpurun_out/strips_small_512_B$B.txt 2>&1
rm -f /tmp/strips_*.npy
done
