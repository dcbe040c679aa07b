cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "C1 - small" "C2 - small"; do
  MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
  MVSK_NO_CHOL=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
done
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_config_parity.py tests/test_golden.py tests/test_gpu_integration.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2m_pytest.log
