cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_op.py fgrad 4 C4 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_c4_fgrad python scripts/prof_op.py fgrad 4 C4 > gpurun_out/ncu_c4_fgrad.log 2>&1
echo "c4 fgrad rc $?"
python scripts/prof_op.py gram 2 C5 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:syrk -s 1 -c 1 -o gpurun_out/prof_c5_gram python scripts/prof_op.py gram 2 C5 > gpurun_out/ncu_c5_gram.log 2>&1
echo "gram rc $?"
ls -la gpurun_out/*.ncu-rep
