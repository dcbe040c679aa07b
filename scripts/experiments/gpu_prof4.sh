cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_op.py hvp8 3 > gpurun_out/p.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 1 -c 1 -o gpurun_out/prof_dmma python scripts/prof_op.py hvp8 3 > gpurun_out/ncu_dmma.log 2>&1
echo "ncu rc $?"
