cd $GRAFT_REPO_ROOT
MVSK_PROFILE=1 timeout 600 python scripts/solve_bench.py --configs C1,C2,C3 --cpu-max-n 0 --reps 2 2>&1 | grep -E "profile|config|C[1-4]" | cut -c1-220 | head -60
