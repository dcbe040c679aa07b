cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/gram_pcg_check.py > gpurun_out/r2_gram_pcg_check.txt 2>&1; echo "rc $?"
cat gpurun_out/r2_gram_pcg_check.txt | cut -c1-400
