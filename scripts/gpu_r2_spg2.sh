cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" "MVSK_SPG_SORT=1"; do
  for cfg in "C4" "C3 20" "C2 -"; do
    echo "== $v $cfg"; env $v MVSK_PROFILE=1 python scripts/one_solve_prof.py $cfg 2>&1 | grep -E "^ok|spg graph" | tail -2
  done
done
timeout 1500 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_solver.py tests/test_gpu_integration.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2o_pytest.log
