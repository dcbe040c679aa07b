cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2_C2s_launches.csv python scripts/one_solve_prof.py C2 - small > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r2_C2s_launches.csv 12
