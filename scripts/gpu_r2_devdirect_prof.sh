cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MVSK_DEVICE_DIRECT=1 MVSK_GPCG_PROF=1
for a in "C2 - small" "C1 - small"; do
  python scripts/one_solve_prof.py $a 2>&1 | grep -E "gdirect|^ok" | (head -3; tail -3)
done
