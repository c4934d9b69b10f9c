mkdir -p gpurun_out
rm -f /tmp/strips_*.npy
for B in 256 4096; do
( PG_STRIPS=0 timeout 900 python tools/probe_strips.py 512 $B; PG_STRIPS=1 timeout 900 python tools/probe_strips.py 512 $B ) > gpurun_out/strips_uout_512_B$B.txt 2>&1
rm -f /tmp/strips_*.npy
done
timeout 900 python -m pytest tests/test_gpu_strips.py -q > gpurun_out/pytest_strips.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strips.log
PINTGPU_GRAPHS=0 timeout 1200 python tools/probe_breakdown.py cfg4 merge > gpurun_out/bd_cfg4_strips3.txt 2>&1
