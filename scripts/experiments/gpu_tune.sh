cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/tune_stream.py C5 hvp8,third8,hvp4 > gpurun_out/tune_c5_cluster.log 2>&1
tail -4 gpurun_out/pytest_gpu.log; cat gpurun_out/tune_c5_cluster.log | tail -40
