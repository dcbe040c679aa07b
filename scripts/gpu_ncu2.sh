cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
python bench.py --steps 3 --warmup 3 --no-extra --no-solve > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-solve > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?"
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 6 -c 1 -o gpurun_out/prof_hvp python bench.py --steps 3 --warmup 3 --no-extra --no-solve > gpurun_out/ncu_full.log 2>&1
echo "full rc $?"
python scripts/prof_op.py third 4 > gpurun_out/p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 1 -o gpurun_out/prof_third2 python scripts/prof_op.py third 4 > gpurun_out/ncu_third2.log 2>&1
echo "third rc $?"
python scripts/prof_op.py gram 2 > gpurun_out/p2.log 2>&1 && ncu --set full --clock-control none -k regex:syrk -s 1 -c 1 -o gpurun_out/prof_gram2 python scripts/prof_op.py gram 2 > gpurun_out/ncu_gram2.log 2>&1
echo "gram rc $?"
tail -1 gpurun_out/plain.log
