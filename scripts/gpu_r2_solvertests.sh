cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_config_parity.py tests/test_golden.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc $?"; tail -6 gpurun_out/r2i_pytest.log
