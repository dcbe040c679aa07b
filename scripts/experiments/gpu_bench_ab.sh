cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export MVSK_DMMA_V1=1; else unset MVSK_DMMA_V1; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-solve 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('v1=$v', d['value'], d['ops']['hvp8_ms'], d['ops']['third_ms'])"
done
unset MVSK_DMMA_V1
timeout 200 python scripts/dmma_ab.py C5 hvp8 pipe,v1 2>&1 | grep " ms\|diff"
