cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python scripts/solve_bench.py --configs C1,C2,C3,C4 --cpu-max-n 800 --reps 3 > gpurun_out/solve_bench.log 2>&1; echo "rc $?" >> gpurun_out/solve_bench.log
cat gpurun_out/solve_bench.log
