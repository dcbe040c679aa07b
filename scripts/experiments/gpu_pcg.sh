cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 3 > gpurun_out/solve_dev.log 2>&1
MVSK_HOST_PCG=1 timeout 900 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 3 > gpurun_out/solve_host.log 2>&1
cut -c1-260 gpurun_out/solve_dev.log; cut -c1-260 gpurun_out/solve_host.log
