cd $GRAFT_REPO_ROOT
python scripts/one_solve.py C4 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster_cg --launch-skip 21 -c 2 -o gpurun_out/prof_ccg python scripts/one_solve.py C4 > gpurun_out/ncu_ccg.log 2>&1; echo "rc $?"
