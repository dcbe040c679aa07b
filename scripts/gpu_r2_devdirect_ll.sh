cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MVSK_DEVICE_DIRECT=1
for a in "C2 - small" "C1 - small"; do
  set -- $a
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2c_$1_devdirect_launches.csv python scripts/one_solve_prof.py $a > /dev/null 2>&1
  python scripts/launch_agg.py gpurun_out/r2c_$1_devdirect_launches.csv 14
done
