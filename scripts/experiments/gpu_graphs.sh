cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 900 python scripts/solve_bench.py --configs C1,C2,C3,C4 --cpu-max-n 0 --reps 3 > gpurun_out/solve_graphs.log 2>&1; echo "rc $?" >> gpurun_out/solve_graphs.log
MVSK_NO_GRAPHS=1 timeout 900 python scripts/solve_bench.py --configs C1,C2,C3,C4 --cpu-max-n 0 --reps 3 > gpurun_out/solve_nographs.log 2>&1; echo "rc $?" >> gpurun_out/solve_nographs.log
tail -30 gpurun_out/solve_graphs.log gpurun_out/solve_nographs.log
