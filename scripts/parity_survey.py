"""Solve-level parity survey: CPU oracle (1 thread), CPU oracle with a different
summation order (2 threads), and the GPU driver, at the default epsilon and a
tight one. Prints status / iterations / x distances / objective gaps."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.datagen import make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

cases = []
for seed in range(4):
    n = 5 + 3 * seed
    A, mu = rh.lcg_panel(n, 60, seed + 7)
    cases.append((f"lcg{seed}", A, mu, rh.crra(4.0 + seed), "small"))
for name, kappa, mode in [("C1", 1.0, "small"), ("C2", 1.0, "small"), ("C2", 10.0, "small"), ("C2", 100.0, "small"),
                          ("C2", 1000.0, "small"), ("C2", 1.0, "large"), ("C2", 10.0, "large"),
                          ("C2", 100.0, "large"), ("C2", 1000.0, "large")]:
    A, mu, c = make_panel(name, seed=11, kappa=kappa)
    cases.append((f"{name}-k{kappa:g}-{mode}", A, mu, c, mode))

for label, A, mu, c, mode in cases:
    for eps in (1e-6, 1e-10):
        res = []
        for who in ("cpu1", "cpu2", "gpu"):
            cfg = po.preset(mode) if who != "gpu" else preset(mode)
            cfg.has_max_elapsed = 0
            cfg.epsilon = eps
            if who == "gpu":
                x, r = GpuOracle(A, mu, c).solve(cfg)
            else:
                po.set_threads(1 if who == "cpu1" else 2)
                x, r = po.solve(A, mu, c, cfg)
                po.set_threads(1)
            res.append((x, r))
        (x1, r1), (x2, r2), (xg, rg) = res
        act = lambda x: tuple(np.nonzero(x <= 1e-8 + 1e-12)[0])
        print(f"{label:18s} eps={eps:.0e} st {r1.status}/{r2.status}/{rg.status} it {r1.iterations}/{r2.iterations}/"
              f"{rg.iterations} |x1-x2|={np.max(np.abs(x1 - x2)):.1e} |x1-xg|={np.max(np.abs(x1 - xg)):.1e} "
              f"df={abs(r1.f_star - rg.f_star):.1e} act={'same' if act(x1) == act(xg) else 'DIFF'} "
              f"kkt {r1.kkt_residual:.1e}/{rg.kkt_residual:.1e}", flush=True)
