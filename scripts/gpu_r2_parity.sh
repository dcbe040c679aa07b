cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_config_parity.py tests/test_golden.py -m gpu -q -rA -p no:cacheprovider -s > gpurun_out/r2b_parity.log 2>&1; echo "rc $?"
grep -E "status|passed|failed|Error" gpurun_out/r2b_parity.log | tail -40
