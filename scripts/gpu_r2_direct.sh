cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "C1 - small" "C2 - small"; do
  MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
  MVSK_NO_DEVICE_DIRECT=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc $?"; tail -8 gpurun_out/r2j_pytest.log
