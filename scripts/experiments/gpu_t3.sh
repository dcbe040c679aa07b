cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tune_stream.py C4 hvp8,third8,hvp4 > gpurun_out/tune_c4_multi.log 2>&1
grep -E "dmma0|=0,0" gpurun_out/tune_c4_multi.log
timeout 600 python scripts/tune_stream.py C3 hvp8,third8 > gpurun_out/tune_c3_multi.log 2>&1
grep -E "dmma0|=0,0" gpurun_out/tune_c3_multi.log
