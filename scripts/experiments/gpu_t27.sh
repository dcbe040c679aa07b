cd $GRAFT_REPO_ROOT
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 third8 2>&1 | grep dmma0
MVSK_TUNE_DMMA_FIX="8,-1" TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 third8 2>&1 | grep dmma0 | sed 's/^/[C=8] /'
timeout 300 python -m pytest tests/test_gpu_oracle.py -q -p no:cacheprovider -k multi_rhs 2>&1 | tail -2
