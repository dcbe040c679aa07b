cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in 0 1 2 4 3 6 7; do for c in C5 C4; do MVSK_DMMA_DBG=$d TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py $c hvp8 2>&1 | grep "dmma0" | sed "s/^/[dbg=$d] /"; done; done > gpurun_out/t8.log
for c in "dmma4,1" "dmma8,1"; do MVSK_TUNE_DMMA=${c#dmma} MVSK_DMMA_DBG=1 TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8 2>&1 | grep "dmma0" | sed "s/^/[$c dbg=1] /"; done >> gpurun_out/t8.log
cat gpurun_out/t8.log
