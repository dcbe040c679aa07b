cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MVSK_PROFILE=1 timeout 600 python scripts/solve_bench.py --configs C1,C2,C3,C4 --cpu-max-n 0 --reps 2 > gpurun_out/solveprof.log 2>&1
echo rc $?
grep -E "profile|gpu_s" gpurun_out/solveprof.log | cut -c1-330 | tail -70
