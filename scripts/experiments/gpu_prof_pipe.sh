cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MVSK_DMMA_DBG=${DBG:-15}
python scripts/prof_op.py hvp8 4 C5 > gpurun_out/p_hvp8.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 2 -c 1 -o gpurun_out/prof_pipe_dbg${MVSK_DMMA_DBG} python scripts/prof_op.py hvp8 4 C5 > gpurun_out/ncu_pipe.log 2>&1
echo "rc $?"
