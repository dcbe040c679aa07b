cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/tune_vs.py C4 > gpurun_out/r2_tune_c4_vs.txt 2>&1; echo "rc $?"
cat gpurun_out/r2_tune_c4_vs.txt
