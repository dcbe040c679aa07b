cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MVSK_GPCG_PROF=1 python scripts/one_solve_prof.py C4 2>&1 | grep -E "gpcg" | tail -1
bash scripts/gpu_r2_prof_solves.sh 2>&1 | grep "^ok"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2q_pytest.log
