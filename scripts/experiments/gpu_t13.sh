cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_oracle.py -q -p no:cacheprovider -k multi_rhs 2>&1 | tail -3
(for t in "4,-1" "8,-1"; do MVSK_TUNE_DMMA_FIX=$t TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C4 hvp8 2>&1 | grep "dmma0" | sed "s/^/[$t] /"; done
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8,third8 2>&1 | grep "dmma0") | tee gpurun_out/t13.log
