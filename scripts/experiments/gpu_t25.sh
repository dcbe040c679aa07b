cd $GRAFT_REPO_ROOT
for r in 1 8 16 32 64; do echo "== min rows $r"; MVSK_MIN_ROWS_PER_CTA=$r ./scripts/_bin/latency_bench 500 20 | grep -v cuda; MVSK_MIN_ROWS_PER_CTA=$r ./scripts/_bin/latency_bench 2500 800 | grep -E "make_cache |hvp"; done
