cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench 2>/dev/null
for s in "500 20" "1000 100"; do echo "== T n = $s"; MVSK_SMALL_PROF=1 ./scripts/_bin/latency_bench $s 2>&1 | grep -v "memcpy\|Synchron"; done
