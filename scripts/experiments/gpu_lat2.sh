cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out scripts/_bin
nvcc -O2 -gencode arch=compute_100a,code=sm_100a scripts/sync_floor.cu -o scripts/_bin/sync_floor && timeout 120 scripts/_bin/sync_floor > gpurun_out/sync_floor.txt 2>&1
cat gpurun_out/sync_floor.txt
MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C1,C2 --cpu-max-n 0 --reps 2 > gpurun_out/solveprof2.log 2>&1
grep -E "profile" gpurun_out/solveprof2.log | cut -c1-400 | awk 'NR%3==0'
