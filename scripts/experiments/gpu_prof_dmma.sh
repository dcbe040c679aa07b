cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_op.py hvp8 4 C5 > gpurun_out/p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 2 -c 1 -o gpurun_out/prof_dmma_c5 python scripts/prof_op.py hvp8 4 C5 > gpurun_out/ncu_d5.log 2>&1
echo "rc $?"
python scripts/prof_op.py hvp8 4 C4 > gpurun_out/p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 2 -c 1 -o gpurun_out/prof_dmma_c4 python scripts/prof_op.py hvp8 4 C4 > gpurun_out/ncu_d4.log 2>&1
echo "rc $?"
