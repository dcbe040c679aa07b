cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gram_ab.py C5 1 0 2>&1 | tail -2
MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C1,C2 --cpu-max-n 0 --reps 2 > gpurun_out/solveprof3.log 2>&1
grep -E "profile" gpurun_out/solveprof3.log | cut -c1-400 | awk 'NR%3==0'
grep -E "gpu_s" gpurun_out/solveprof3.log | cut -c1-200
