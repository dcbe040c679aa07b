cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(TUNE_DEFAULT_ONLY=1 timeout 600 python scripts/tune_stream.py C5 hvp8,third8,hvp1
 TUNE_DEFAULT_ONLY=1 timeout 600 python scripts/tune_stream.py C4 hvp8,third8,hvp1,third) > gpurun_out/t7.log 2>&1
cat gpurun_out/t7.log
bash scripts/gpu_tests.sh
