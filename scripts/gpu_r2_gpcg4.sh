cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MVSK_GPCG_PROF=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py C4 2>&1 | grep -E "mvsk profile|^ok|gpcg" | tail -4
MVSK_GPCG_PROF=1 python scripts/one_solve_prof.py C3 20 2>&1 | grep -E "gpcg" | tail -2
MVSK_GPCG_PROF=1 python scripts/one_solve_prof.py C2 - large 2>&1 | grep -E "gpcg" | tail -2
timeout 900 python scripts/gram_pcg_check.py 2>&1 | cut -c1-300
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2g_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -6 gpurun_out/r2g_pytest_gpu.log
