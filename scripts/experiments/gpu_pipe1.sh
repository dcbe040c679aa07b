cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_oracle.py -x -q -k "multi_rhs or graph or group or device" > gpurun_out/pt_pipe.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pt_pipe.log
timeout 300 python scripts/dmma_ab.py C5 hvp8,third8,hvp4,third4 pipe,v1 2>&1 | tail -20
timeout 300 python scripts/dmma_ab.py C5 third8,hvp8 pipeC8,pipeC4,v1 2>&1 | tail -20
timeout 300 python scripts/dmma_ab.py C4 hvp8,third8 pipe,v1 2>&1 | tail -20
