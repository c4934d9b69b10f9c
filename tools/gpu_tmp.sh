mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q -x --deselect "tests/test_gpu_full.py::test_config5_phi_matches_oracle" ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
