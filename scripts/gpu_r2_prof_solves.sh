cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "C4 - large" "C3 20 large" "C3 5 large" "C2 - small" "C1 - small" "C2 - large"; do
  MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -3
done > gpurun_out/r2_solve_profiles.txt 2>&1
cat gpurun_out/r2_solve_profiles.txt
