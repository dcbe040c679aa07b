cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin gpurun_out
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench 2>/dev/null
for s in "500 20" "1000 100"; do echo "== T n = $s"; ./scripts/_bin/latency_bench $s | grep -v "memcpy\|Synchron"; done
bash scripts/gpu_r2_prof_solves.sh 2>&1 | grep "^ok"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc $?"; tail -6 gpurun_out/r2q_pytest.log
