cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_op.py gram 2 > gpurun_out/p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:syrk_dmma -s 1 -c 1 -o gpurun_out/prof_gram python scripts/prof_op.py gram 2 > gpurun_out/ncu_gram.log 2>&1
echo "ncu rc $?"
