"""Does a solve depend on what ran before it on the same GpuOracle? (debugging
aid for the stress-profile case: directions at a point, then solve)"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset, tangent_config  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

n, T, seed = 12, 80, 1
c = np.array([10.0, 1, 10, 1])
A, mu = rh.lcg_panel(n, T, seed + 31)
x = rh.simplex_point(n, seed + 3, 1e-6)
cfg = preset("small")
cfg.has_max_elapsed = 0
cfg.epsilon = 1e-10
ccfg = po.preset("small")
ccfg.has_max_elapsed = 0
ccfg.epsilon = 1e-10
xc, rc = po.solve(A, mu, c, ccfg)
modes = [("direct", 0.0), ("direct", 1e-6), ("pcg", 1e-4)]
for pre_ops in ([], [0], [1], [2], [0, 1], [0, 1, 2], "cache"):
    g = GpuOracle(A, mu, c)
    if pre_ops == "cache":
        gc = g.make_cache(x)
    else:
        gc = g.make_cache(x) if pre_ops else None
        for k in pre_ops:
            m, lam = modes[k]
            g.yand_direction(gc, tangent_config(m, lam=lam), seed)
    xs, rs = g.solve(cfg)
    print(pre_ops, "status", rs.status, "it", rs.iterations, "faces", rs.face_events, "restarts", rs.restarts,
          "dx", float(np.max(np.abs(xs - xc))), flush=True)
    # and a second solve on the same oracle
    xs2, rs2 = g.solve(cfg)
    print("   again: status", rs2.status, "dx", float(np.max(np.abs(xs2 - xc))), flush=True)
    g.close()
