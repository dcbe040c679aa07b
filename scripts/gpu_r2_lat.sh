cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench || exit 1
for s in "500 20" "1000 100" "5000 5000"; do echo "== T n = $s"; ./scripts/_bin/latency_bench $s; done
