cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 900 python scripts/solve_bench.py --configs C2,C3,C4 --cpu-max-n 0 --reps 3 2>&1 | cut -c1-150
