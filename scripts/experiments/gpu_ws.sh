cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python scripts/dmma_ab.py C5 hvp8,third8,hvp4,third4 ws,pipe,v1 2>&1 | grep " ms\|diff\|rror"
MVSK_DMMA_WS=1 timeout 600 python -m pytest tests/test_gpu_oracle.py -x -q -k "multi_rhs or graph or group or device" 2>&1 | tail -2
