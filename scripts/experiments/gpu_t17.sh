cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 0 1; do for d in "4,1" "4,-1"; do
MVSK_DMMA_EARLY=$e MVSK_TUNE_DMMA_FIX=$d TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp8 2>&1 | grep dmma0 | sed "s/^/[early=$e D=$d] /"
done; done
for e in 0 1; do MVSK_DMMA_EARLY=$e TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 third8 2>&1 | grep dmma0 | sed "s/^/[early=$e] /"; MVSK_DMMA_EARLY=$e TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C4 hvp8,third8 2>&1 | grep dmma0 | sed "s/^/[early=$e] /"; done
