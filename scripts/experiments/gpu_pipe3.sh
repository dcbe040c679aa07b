cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_oracle.py -x -q -k "multi_rhs or graph or group or device" 2>&1 | tail -2
timeout 200 python scripts/dmma_ab.py C5 hvp8,third8,hvp4,third4 pipe,v1 2>&1 | grep " ms\|diff"
