cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
(TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8,third8; TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C4 hvp8,third8) 2>&1 | grep dmma0
