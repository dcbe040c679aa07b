cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pf in 0 2 3 4 6 8; do for c in C5 C4; do MVSK_DMMA_PF=$pf TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py $c hvp8,third8 2>&1 | grep "dmma0" | sed "s/^/[pf=$pf] /"; done; done > gpurun_out/t9.log
cat gpurun_out/t9.log
