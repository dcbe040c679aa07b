cd $GRAFT_REPO_ROOT
./scripts/_bin/sync_floor
LD_LIBRARY_PATH=paper_2604_25378_b200/_build ./scripts/_bin/latency_bench 500 20 | grep -v cuda
LD_LIBRARY_PATH=paper_2604_25378_b200/_build ./scripts/_bin/latency_bench 1000 100 | grep -v cuda
