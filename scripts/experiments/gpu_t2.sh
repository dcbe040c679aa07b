cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for c in C2 C3 C4; do timeout 600 python scripts/tune_stream.py $c hvp1,fgrad,lines > gpurun_out/tune_$c.log 2>&1; grep default gpurun_out/tune_$c.log; for op in hvp1 fgrad lines; do grep " $op Q" gpurun_out/tune_$c.log | sort -t: -k2 -n | head -1; done; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
