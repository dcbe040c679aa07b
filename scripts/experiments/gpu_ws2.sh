cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 300 python scripts/dmma_ab.py C5 hvp8,hvp4,third4,third8 ws,pipe,v1 2>&1 | grep " ms\|diff\|rror" > gpurun_out/ab.txt; cat gpurun_out/ab.txt
timeout 300 python scripts/dmma_ab.py C4 hvp8,third8 ws,v1 2>&1 | grep " ms\|diff\|rror"
python scripts/prof_op.py hvp8 4 C5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_dmma -s 2 -c 1 -o gpurun_out/prof_ws_hvp8_c5 python scripts/prof_op.py hvp8 4 C5 > gpurun_out/ncu_ws.log 2>&1; echo "ncu rc $?"
