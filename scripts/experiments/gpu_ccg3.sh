cd $GRAFT_REPO_ROOT
MVSK_CCG_PROF=1 timeout 120 python scripts/one_solve.py C4 2>&1 | tail -3
MVSK_CCG_PROF=1 timeout 120 python scripts/one_solve.py C3 2>&1 | tail -3
