cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin gpurun_out
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench 2>/dev/null
for s in "500 20" "1000 100" "5000 5000"; do echo "== T n = $s"; ./scripts/_bin/latency_bench $s; done
timeout 900 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_integration.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
bash scripts/gpu_r2_prof_solves.sh 2>&1 | grep "^ok"
