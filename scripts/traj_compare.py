"""Observer trajectories of one solve on the GPU and on the CPU parity oracle
(bit-identical to the reference build), side by side, to locate the first
iteration where they part (debugging aid)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lcg_n9_T60"
pre = sys.argv[2] if len(sys.argv) > 2 else "small"
if name.startswith("lcg:"):  # lcg:n:T:seed:c1,c2,c3,c4 (tests/refhelpers.lcg_panel)
    from tests import refhelpers as rh
    _, n_, T_, s_, cs = name.split(":")
    A_, mu_ = rh.lcg_panel(int(n_), int(T_), int(s_))
    g = {"A": A_, "mu": mu_, "c": np.array([float(v) for v in cs.split(",")])}
else:
    g = dict(np.load(ROOT / "tests" / "golden" / f"{name}.npz"))
cfg_g, cfg_c = preset(pre), po.preset(pre)
for c in (cfg_g, cfg_c):
    c.has_max_elapsed = 0
    c.epsilon = 1e-10
tg, tc = [], []
xg, rg = GpuOracle(g["A"], g["mu"], g["c"]).solve(cfg_g, observer=lambda i, f, x: tg.append((i, f, x)))
xc, rc = po.solve(g["A"], g["mu"], g["c"], cfg_c, observer=lambda i, f, x: tc.append((i, f, x)))
print("gpu", rg.status, rg.iterations, rg.face_events, rg.restarts, rg.kkt_residual, "cpu", rc.status, rc.iterations,
      rc.face_events, rc.restarts, rc.kkt_residual)
print("final dx", float(np.max(np.abs(xg - xc))))
np.set_printoptions(precision=17, linewidth=200)
for k in range(max(len(tg), len(tc))):
    a = tg[k] if k < len(tg) else None
    b = tc[k] if k < len(tc) else None
    dx = float(np.max(np.abs(a[2] - b[2]))) if a and b and a[2].size == b[2].size else float("nan")
    print(k, a[:2] if a else None, b[:2] if b else None, f"dx {dx:.3e}")
    if a and b and dx > 1e-9:
        print(" gpu x", a[2])
        print(" cpu x", b[2])
        if k > 0:
            print(" prev x", tc[k - 1][2])
        break
