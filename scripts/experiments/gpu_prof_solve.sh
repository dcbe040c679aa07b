cd $GRAFT_REPO_ROOT
MVSK_PROFILE=1 timeout 900 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 1 2>&1 | grep -E "profile|config" | cut -c1-250
