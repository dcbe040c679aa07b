cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/one_solve.py C4 > gpurun_out/one_solve.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/one_solve.py C4 > gpurun_out/ncu_c4.log 2>&1
echo "rc $?"; cat gpurun_out/one_solve.log; tail -2 gpurun_out/ncu_c4.log
