cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TUNE_DEFAULT_ONLY=1 timeout 600 python scripts/tune_stream.py C5 hvp1,hvp2,third,fgrad,lines > gpurun_out/t5.log 2>&1
for t in "8,1,2,2,1" "8,1,2,3,1" "8,1,1,4,1"; do MVSK_TUNE=$t TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 third,hvp2 2>&1 | sed "s/^/[$t] /" >> gpurun_out/t5.log; done
cat gpurun_out/t5.log
bash scripts/gpu_tests.sh
