cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-600
python scripts/prof_op.py hvp8 3 > gpurun_out/p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_cluster -s 1 -c 1 -o gpurun_out/prof_hvp8 python scripts/prof_op.py hvp8 3 > gpurun_out/ncu_hvp8.log 2>&1
echo "ncu rc $?"
