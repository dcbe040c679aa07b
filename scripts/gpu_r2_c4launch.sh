cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MVSK_PROFILE=1 python scripts/one_solve_prof.py C4 2>&1 | grep -E "mvsk profile|^ok" | tail -2
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_solve_launches.csv python scripts/one_solve_prof.py C4 > /dev/null 2>&1
echo "ncu rc $?"
python scripts/launch_agg.py gpurun_out/r2_c4_solve_launches.csv | head -30
