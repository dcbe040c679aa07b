cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?"
python bench.py --steps 3 --warmup 3 --no-extra --no-solve > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-solve > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?"
python scripts/one_solve_prof.py C4 > /dev/null 2>&1 && \
timeout 900 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches_warm.csv python scripts/one_solve_prof.py C4 > /dev/null 2>&1
echo "c4 launch list rc $?"
