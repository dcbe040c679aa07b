cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider -k "spg" > gpurun_out/pytest_spg.log 2>&1; echo "spg tests rc $?"; tail -15 gpurun_out/pytest_spg.log
MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C1,C2 --cpu-max-n 0 --reps 3 > gpurun_out/solveprof5.log 2>&1
grep -E "profile" gpurun_out/solveprof5.log | cut -c1-330 | awk 'NR%4==0'
grep -E "gpu_s" gpurun_out/solveprof5.log | cut -c1-170
