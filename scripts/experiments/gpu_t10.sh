cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for t in "4,1" "4,-1"; do MVSK_DMMA_PF=0 MVSK_TUNE_DMMA_FIX=$t TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8,third8 2>&1 | grep "dmma0" | sed "s/^/[$t] /"; done > gpurun_out/t10.log
for t in "8,1" "8,-1"; do MVSK_DMMA_PF=0 MVSK_TUNE_DMMA_FIX=$t TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C4 hvp8,third8 2>&1 | grep "dmma0" | sed "s/^/[$t] /"; done >> gpurun_out/t10.log
cat gpurun_out/t10.log
