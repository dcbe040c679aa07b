cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/r2k_bench.log | cut -c1-600
python scripts/one_solve_prof.py C4 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2k_c4_solve_launches.csv python scripts/one_solve_prof.py C4 > gpurun_out/r2k_c4_ok.txt 2>&1
python scripts/launch_agg.py gpurun_out/r2k_c4_solve_launches.csv | head -16
python scripts/one_solve_prof.py C4
