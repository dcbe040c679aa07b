"""Print CPU-oracle vs GPU solver trajectories side by side (observer records)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset, tangent_config  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n = 5 + 3 * seed
A, mu = rh.lcg_panel(n, 60, seed + 7)
c = rh.crra(4.0 + seed)
tc, tg = [], []
xc, rc = po.solve(A, mu, c, po.preset("small"), observer=lambda it, f, x: tc.append((it, f, x)))
gpu = GpuOracle(A, mu, c)
xg, rg = gpu.solve(preset("small"), observer=lambda it, f, x: tg.append((it, f, x)))
print("cpu iters", rc.iterations, "gpu iters", rg.iterations, "status", rc.status, rg.status)
for k in range(max(len(tc), len(tg))):
    a = tc[k] if k < len(tc) else None
    b = tg[k] if k < len(tg) else None
    if a and b:
        print(k, a[0], b[0], f"{a[1]:.17g} {b[1]:.17g} dx={np.max(np.abs(a[2]-b[2])):.3e}")
    else:
        print(k, a and a[:2], b and b[:2])
# direction at the start point, direct mode, CPU vs GPU
x0 = np.full(n, 1.0 / n)
co = po.CpuOracle(A, mu, c)
cc = co.make_cache(x0)
gc = gpu.make_cache(x0)
dc, _ = co.yand_direction(cc, po.tangent_config("direct"), 1)
dg, _ = gpu.yand_direction(gc, tangent_config("direct"), 1)
print("dir diff at x0", np.max(np.abs(dc - dg)), np.max(np.abs(dc)))
lc = co.line_model(cc, dc, 1.0)
lg = gpu.line_model(gc, dc, 1.0)
print("line model cpu", lc[:5])
print("line model gpu", [lg.a0, lg.a1, lg.a2, lg.a3, lg.a4])
