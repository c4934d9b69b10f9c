mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_full.py::test_nonlinear_config3_n64_matches_reference_engine tests/test_gpu_mgrit.py tests/test_gpu_phi.py tests/test_gpu_edge.py tests/test_gpu_multirank.py -q > gpurun_out/pytest_nk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nk.log
timeout 900 python tools/probe_cfg3.py 16384 profile > gpurun_out/cfg3_jac.txt 2>&1
PG_NK_JAC=0 timeout 900 python tools/probe_cfg3.py 16384 > gpurun_out/cfg3_nojac.txt 2>&1
timeout 600 python tools/probe_breakdown.py cfg2 > gpurun_out/bd_cfg2.txt 2>&1
PINTGPU_GRAPHS=0 timeout 600 python tools/probe_breakdown.py cfg2 > gpurun_out/bd_cfg2_nograph.txt 2>&1
PG_RB_ALT=2 timeout 600 python tools/probe_band.py cfg4 0:4096 1:256 > gpurun_out/probe_band_cfg4_alt2.txt 2>&1
timeout 600 python tools/probe_band.py cfg4 0:4096 1:256 > gpurun_out/probe_band_cfg4_alt0.txt 2>&1
