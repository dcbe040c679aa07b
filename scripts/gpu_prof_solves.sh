# Per-solve host timing breakdown (MVSK_PROFILE) of the BASELINE solve configs, plus the per-phase
# clock64 profiles of the reduced-Hessian PCG / direct cluster kernels (MVSK_GPCG_PROF):
#   gpurun -- 'bash scripts/gpu_prof_solves.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for a in "C4 - large" "C3 20 large" "C3 5 large" "C2 - small" "C1 - small" "C2 - large"; do
  MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
done
for a in "C4 - large" "C3 20 large" "C2 - small"; do
  MVSK_GPCG_PROF=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "gpcg|gdirect|^ok" | (head -2; tail -3)
done
} > gpurun_out/solve_profiles.txt 2>&1
cat gpurun_out/solve_profiles.txt
