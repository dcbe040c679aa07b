cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_op.py third 4 > gpurun_out/p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 1 -o gpurun_out/prof_third python scripts/prof_op.py third 4 > gpurun_out/ncu_third.log 2>&1
echo "rc $?"; tail -3 gpurun_out/ncu_third.log
