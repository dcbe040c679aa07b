cd $GRAFT_REPO_ROOT
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8 2>&1 | grep dmma0
MVSK_DMMA_OCC2=1 TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8 2>&1 | grep dmma0 | sed 's/^/[occ2] /'
MVSK_DMMA_OCC2=1 timeout 300 python -m pytest tests/test_gpu_oracle.py -q -p no:cacheprovider -k multi_rhs 2>&1 | tail -2
