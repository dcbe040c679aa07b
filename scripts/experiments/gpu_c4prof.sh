cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "direct or gram or solve" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
python scripts/one_solve_prof.py C4 && \
timeout 900 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches_warm.csv python scripts/one_solve_prof.py C4 > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/c4_launches_warm.csv 30
MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C1,C2 --cpu-max-n 0 --reps 2 > gpurun_out/solveprof3.log 2>&1
grep -E "profile" gpurun_out/solveprof3.log | cut -c1-400 | awk 'NR%3==0' | head -2
