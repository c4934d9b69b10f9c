mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_full.py::test_nonlinear_config3_n64_matches_reference_engine tests/test_gpu_mgrit.py tests/test_gpu_phi.py::test_nonlinear_newton_phi_matches_oracle tests/test_gpu_edge.py -x -q > gpurun_out/pytest_nk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nk.log
timeout 900 python tools/probe_cfg3.py 16384 profile > gpurun_out/cfg3_new.txt 2>&1
PG_NK_BURST=1 timeout 900 python tools/probe_cfg3.py 16384 > gpurun_out/cfg3_burst1.txt 2>&1
