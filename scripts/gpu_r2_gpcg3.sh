cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MVSK_GPCG_PROF=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py C4 2>&1 | grep -E "mvsk profile|^ok|gpcg" | tail -8
MVSK_GPCG_PROF=1 python scripts/one_solve_prof.py C3 20 2>&1 | grep -E "gpcg" | tail -3
MVSK_GPCG_PROF=1 python scripts/one_solve_prof.py C2 - large 2>&1 | grep -E "gpcg" | tail -3
