cd $GRAFT_REPO_ROOT
for v in "" 1; do
echo "== MVSK_NO_CG_TAIL=$v"
if [ -z "$v" ]; then unset MVSK_NO_CG_TAIL; else export MVSK_NO_CG_TAIL=1; fi
MVSK_PROFILE=1 timeout 900 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 1 2>&1 | grep -E "profile|config" | cut -c1-140 | awk 'NR%2==0 || /config/' | tail -6
done
python - <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2604_25378_b200.datagen import make_panel
from paper_2604_25378_b200.gpu_oracle import GpuOracle, tangent_config
from tests import refhelpers as rh
A, mu, c = make_panel("C3", seed=11)
g = GpuOracle(A, mu, c)
x = rh.simplex_point(A.shape[1], 3, 1e-6)
for i in range(4):
    gc = g.make_cache(x)
    l0 = g.launch_count()
    d, diag = g.yand_direction(gc, tangent_config("pcg", lam=1e-4), 7)
    print("direction", i, "launches", g.launch_count() - l0, "krylov", diag.krylov_iters)
PY
