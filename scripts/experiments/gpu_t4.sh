cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for c in C2 C3 C4; do timeout 600 python scripts/tune_stream.py $c hvp1,fgrad,lines > gpurun_out/tune_$c.log 2>&1; grep default gpurun_out/tune_$c.log; for op in hvp1 fgrad lines; do grep " $op Q" gpurun_out/tune_$c.log | sort -t: -k2 -n | head -1; done; done
timeout 600 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 3 2>&1 | cut -c1-200
