"""GPU vs CPU final weights at several epsilons (solve parity diagnostics)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.datagen import make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

for name, kappa, mode in [("C1", 1.0, "small"), ("C2", 1.0, "small"), ("C2", 10.0, "small"), ("C2", 100.0, "small"),
                          ("C2", 1000.0, "small"), ("C2", 1.0, "large"), ("C2", 10.0, "large"),
                          ("C2", 100.0, "large"), ("C2", 1000.0, "large")]:
    A, mu, c = make_panel(name, seed=11, kappa=kappa)
    g = GpuOracle(A, mu, c)
    for eps in (1e-10, 1e-12):
        cc, cg = po.preset(mode), preset(mode)
        for cfg in (cc, cg):
            cfg.has_max_elapsed = 0
            cfg.epsilon = eps
        xc, rc = po.solve(A, mu, c, cc)
        xg, rg = g.solve(cg)
        print(f"{name} k={kappa:g} {mode} eps={eps:g}: cpu st={rc.status} kkt={rc.kkt_residual:.1e} it={rc.iterations} | "
              f"gpu st={rg.status} kkt={rg.kkt_residual:.1e} it={rg.iterations} | dx={np.max(np.abs(xg - xc)):.1e} "
              f"df={abs(rg.f_star - rc.f_star):.1e}", flush=True)
