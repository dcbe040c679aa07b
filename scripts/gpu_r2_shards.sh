cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -rA -p no:cacheprovider -x > gpurun_out/r2c_shards.log 2>&1; echo "shards rc $?"
grep -E "passed|failed|^E |Error" gpurun_out/r2c_shards.log | head -30
timeout 600 python scripts/debug_golden_case.py lcg_n9_T60 > gpurun_out/r2c_lcg_debug.log 2>&1; echo "debug rc $?"
cat gpurun_out/r2c_lcg_debug.log | cut -c1-700
