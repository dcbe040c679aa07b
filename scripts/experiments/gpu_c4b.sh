cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
MVSK_CCG_PROF=1 python scripts/one_solve_prof.py C4 2>&1 | tail -2
timeout 900 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches_warm.csv python scripts/one_solve_prof.py C4 > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/c4_launches_warm.csv 16
MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 3 > gpurun_out/solveprof4.log 2>&1
grep -E "gpu_s" gpurun_out/solveprof4.log | cut -c1-200
