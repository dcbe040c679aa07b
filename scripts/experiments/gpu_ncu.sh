cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
# launch list of the bench's timed region (plain run first, then ncu)
python bench.py --steps 3 --warmup 3 --no-extra > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extra > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?"
python bench.py --steps 3 --warmup 3 --no-extra > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 6 -c 1 -o gpurun_out/prof_hvp python bench.py --steps 3 --warmup 3 --no-extra > gpurun_out/ncu_full.log 2>&1
echo "full rc $?"
tail -3 gpurun_out/ncu_full.log
