cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "C4 - large" "C2 - small" "C1 - small"; do  # gpurun -- "bash scripts/gpu_launch_lists.sh"
  set -- $a
  MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "^ok" | tail -1
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2_$1_solve_launches.csv python scripts/one_solve_prof.py $a > /dev/null 2>&1
  python scripts/launch_agg.py gpurun_out/r2_$1_solve_launches.csv 14
done
