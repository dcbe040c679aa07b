"""small-preset solve then large-preset solve on one GpuOracle (debugging aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

A, mu = rh.lcg_panel(12, 80, 32)
c = np.array([10.0, 1, 10, 1])
order = sys.argv[1].split(",") if len(sys.argv) > 1 else ["small", "large"]
g = GpuOracle(A, mu, c)
held = g.make_cache(rh.simplex_point(12, 4, 1e-6)) if "--hold" in sys.argv else None
for pre in order:
    cfg = preset(pre)
    cfg.has_max_elapsed = 0
    cfg.epsilon = 1e-10
    ccfg = po.preset(pre)
    ccfg.has_max_elapsed = 0
    ccfg.epsilon = 1e-10
    tr = []
    xg, rg = g.solve(cfg, observer=lambda i, f, x: tr.append((i, f)))
    xc, rc = po.solve(A, mu, c, ccfg)
    print(pre, "gpu", rg.status, rg.iterations, rg.restarts, "cpu", rc.status, rc.iterations,
          "dx %.2e" % float(np.max(np.abs(xg - xc))), tr[:12], flush=True)
