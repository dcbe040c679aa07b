cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for op in hvp8 third8; do
python scripts/prof_op.py $op 4 C5 > gpurun_out/p_$op.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 2 -c 1 -o gpurun_out/prof_${op}_c5 python scripts/prof_op.py $op 4 C5 > gpurun_out/ncu_$op.log 2>&1
echo "$op rc $?"
done
