cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_op.py fgrad 4 C4 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r2_c4_fgrad python scripts/prof_op.py fgrad 4 C4 > gpurun_out/r2_ncu_c4_fgrad.log 2>&1
echo "c4 fgrad rc $?"
python scripts/prof_op.py hvp8 3 C5 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 2 -c 1 -o gpurun_out/r2_c5_hvp8 python scripts/prof_op.py hvp8 3 C5 > gpurun_out/r2_ncu_c5_hvp8.log 2>&1
echo "hvp8 rc $?"
python scripts/prof_op.py hvp1 4 C5 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r2_c5_hvp1 python scripts/prof_op.py hvp1 4 C5 > gpurun_out/r2_ncu_c5_hvp1.log 2>&1
echo "hvp1 rc $?"
ls -la gpurun_out/*.ncu-rep
