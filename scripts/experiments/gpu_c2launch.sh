cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
python scripts/one_solve_prof.py C2 - small && \
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2small_launches.csv python scripts/one_solve_prof.py C2 - small > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/c2small_launches.csv
MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C1,C2 --cpu-max-n 0 --reps 2 > gpurun_out/solveprof3.log 2>&1
grep -E "profile" gpurun_out/solveprof3.log | cut -c1-400 | awk 'NR%3==0' | head -2
grep -E "gpu_s" gpurun_out/solveprof3.log | cut -c1-140
