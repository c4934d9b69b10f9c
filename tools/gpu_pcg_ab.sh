# streamed PCG A/B against the previous build (bitwise + timing)
mkdir -p gpurun_out
L=gpurun_out/pcg_ab.log
: > $L
BASE=$PWD/paper_1912_03106_b200/lib/libpintgpu_base.so
timeout 600 python -m pytest tests/test_gpu_phi.py -x -q > gpurun_out/pcg_tests.log 2>&1; tail -2 gpurun_out/pcg_tests.log >> $L
PINTGPU_LIB=$BASE timeout 300 python tools/probe_pcg_bits.py gpurun_out/pcg_base.npz >> $L 2>&1
timeout 300 python tools/probe_pcg_bits.py gpurun_out/pcg_new.npz >> $L 2>&1
python -c "
import numpy as np
a=np.load('gpurun_out/pcg_base.npz'); b=np.load('gpurun_out/pcg_new.npz')
for k in a.files: print(k, 'identical' if np.array_equal(a[k], b[k]) else 'DIFFERENT')
" >> $L 2>&1
for r in 1 2; do
echo "== base" >> $L
PINTGPU_LIB=$BASE timeout 300 python tools/probe_cfg5.py 1024 >> $L 2>&1
echo "== new" >> $L
timeout 300 python tools/probe_cfg5.py 1024 >> $L 2>&1
done
