cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_default.log
tail -2 gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/bench_ref.log
tail -2 gpurun_out/bench_ref.log
