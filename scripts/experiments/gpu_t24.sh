cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/one_solve_prof.py C4 > gpurun_out/os.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4b_launches.csv python scripts/one_solve_prof.py C4 > gpurun_out/ncu_c4b.log 2>&1
echo "rc $?"; cat gpurun_out/os.log
