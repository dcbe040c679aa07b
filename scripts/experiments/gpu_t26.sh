cd $GRAFT_REPO_ROOT
echo "== default"; ./scripts/_bin/latency_bench 500 20 | grep -v cuda
echo "== no fused"; MVSK_NO_FUSED_FINISH=1 ./scripts/_bin/latency_bench 500 20 | grep -v cuda
echo "== no graphs"; MVSK_NO_GRAPHS=1 ./scripts/_bin/latency_bench 500 20 | grep -v cuda
echo "== no graphs no fused"; MVSK_NO_GRAPHS=1 MVSK_NO_FUSED_FINISH=1 ./scripts/_bin/latency_bench 500 20 | grep -v cuda
