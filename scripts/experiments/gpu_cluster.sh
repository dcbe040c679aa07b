cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "cluster or hvp_third" > gpurun_out/pytest_cluster.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_cluster.log
tail -3 gpurun_out/pytest_cluster.log
timeout 300 python scripts/tune_stream.py C5 hvp8,third8,hvp4 > gpurun_out/tune_c5_cluster.log 2>&1
cat gpurun_out/tune_c5_cluster.log
