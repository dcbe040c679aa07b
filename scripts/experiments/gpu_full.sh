cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python scripts/solve_bench.py --configs C1,C2,C3,C4 --cpu-max-n 800 --reps 3 > gpurun_out/solve_bench.log 2>&1; echo "rc $?" >> gpurun_out/solve_bench.log
cut -c1-330 gpurun_out/solve_bench.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
