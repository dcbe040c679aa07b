cd $GRAFT_REPO_ROOT
timeout 300 python scripts/dmma_ab.py C5 third8,hvp8 ws,v1 2>&1 | grep " ms\|diff\|rror"
timeout 600 python -m pytest tests/test_gpu_oracle.py -x -q -k "multi_rhs" 2>&1 | tail -2
