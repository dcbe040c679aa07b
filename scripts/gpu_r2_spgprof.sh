cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MVSK_PROFILE=1 python scripts/one_solve_prof.py C4 2>&1 | grep -E "mvsk profile|^ok|spg graph" | tail -3
MVSK_PROFILE=1 python scripts/one_solve_prof.py C3 20 2>&1 | grep -E "mvsk profile|^ok|spg graph" | tail -3
timeout 900 python -m pytest tests/test_gpu_solver.py -m gpu -q -p no:cacheprovider -rf -k "stress" > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2n_pytest.log
