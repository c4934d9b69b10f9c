# uniform-1/dt fast path of the streamed PCG: bitwise + timing A/B against the previous build
mkdir -p gpurun_out
L=gpurun_out/pcg_ab.log
: > $L
BASE=$PWD/paper_1912_03106_b200/lib/libpintgpu_base.so
timeout 900 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py tests/test_gpu_edge.py -x -q > gpurun_out/pcg_tests.log 2>&1; tail -2 gpurun_out/pcg_tests.log >> $L
PINTGPU_LIB=$BASE timeout 300 python tools/probe_pcg_bits.py gpurun_out/pcg_base.npz >> $L 2>&1
timeout 300 python tools/probe_pcg_bits.py gpurun_out/pcg_new.npz >> $L 2>&1
python -c "
import numpy as np
a=np.load('gpurun_out/pcg_base.npz'); b=np.load('gpurun_out/pcg_new.npz')
for k in a.files: print(k, 'identical' if np.array_equal(a[k], b[k]) else 'DIFFERENT max %g' % np.max(np.abs(a[k]-b[k])))
" >> $L 2>&1
echo "== base" >> $L
PINTGPU_LIB=$BASE timeout 300 python tools/probe_cfg5.py 256 1024 4096 >> $L 2>&1
echo "== new" >> $L
timeout 300 python tools/probe_cfg5.py 256 1024 4096 >> $L 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sdir --launch-skip 20 -c 1 -o gpurun_out/sdir_full python tools/probe_cfg5.py 1024 > gpurun_out/ncu_sdir.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_supd --launch-skip 20 -c 1 -o gpurun_out/supd_full python tools/probe_cfg5.py 1024 > gpurun_out/ncu_supd.log 2>&1
