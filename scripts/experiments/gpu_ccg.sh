cd $GRAFT_REPO_ROOT
timeout 120 python scripts/one_solve.py C4; echo "c4 rc $?"
timeout 120 python scripts/one_solve.py C3; echo "c3 rc $?"
timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_golden.py -x -q -m gpu 2>&1 | tail -15
for v in 0 1; do
  if [ $v = 1 ]; then export MVSK_NO_CCG=1; else unset MVSK_NO_CCG; fi
  echo "== MVSK_NO_CCG=$v"
  timeout 300 python scripts/solve_bench.py --configs C2,C3,C4 --cpu-max-n 0 --reps 3 2>&1 | grep -E "config" | python3 -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['kappa'], d.get('gamma'), d['preset'], round(d['gpu_s']*1e3,2), 'ms iters', d['gpu_iters'], 'f', d['f'])"
done
