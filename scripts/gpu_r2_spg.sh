cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "C4 -" "C3 20" "C3 5"; do
  MVSK_GPCG_PROF=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok|gpcg" | tail -3
  MVSK_NO_SPG_GRAPH=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
done
timeout 900 python scripts/gram_pcg_check.py 2>&1 | cut -c1-300
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2h_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -6 gpurun_out/r2h_pytest_gpu.log
