"""Robustness sweep of the large preset (cluster SPG preamble on narrow panels)
against the CPU oracle over seeds and kappas: status, active set, |dx|, df.
python scripts/spg_sweep.py [nseeds]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.datagen import make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
bad = 0
for name in ("C1", "C2"):
    for kappa in ((1.0,) if name == "C1" else (1.0, 10.0, 100.0, 1000.0)):
        for seed in range(nseeds):
            A, mu, c = make_panel(name, seed=seed, kappa=kappa)
            cfg, cc = preset("large"), po.preset("large")
            cfg.has_max_elapsed = cc.has_max_elapsed = 0
            cfg.epsilon = cc.epsilon = 1e-10
            g = GpuOracle(A, mu, c)
            xg, rg = g.solve(cfg)
            g.close()
            xc, rc = po.solve(A, mu, c, cc)
            tau = cfg.tau
            same_act = np.array_equal(xg <= tau + 1e-12, xc <= tau + 1e-12)
            dx = float(np.max(np.abs(xg - xc)))
            df = abs(rg.f_star - rc.f_star) / (1 + abs(rc.f_star))
            ok = rg.status == rc.status and same_act and df <= 1e-12
            bad += 0 if ok else 1
            print(f"{name} kappa {kappa:6.0f} seed {seed}: status {rg.status}/{rc.status} ident {rg.identification_steps:3d}/"
                  f"{rc.identification_steps:3d} act {'=' if same_act else 'DIFF'} dx {dx:.1e} df {df:.1e} {'ok' if ok else 'CHECK'}",
                  flush=True)
print("cases needing a look:", bad)
