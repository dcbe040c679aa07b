cd $GRAFT_REPO_ROOT
timeout 900 python scripts/tune_stream.py C5 hvp2 > gpurun_out/t29.log 2>&1
sort -t: -k2 -n gpurun_out/t29.log | head -8; grep default gpurun_out/t29.log
