"""One large-preset case three ways: GPU (default), CPU oracle 1 and 2 threads:
python scripts/case_check.py C2 100 2"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.datagen import make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

name, kappa, seed = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
A, mu, c = make_panel(name, seed=seed, kappa=kappa)
cfg, cc = preset("large"), po.preset("large")
cfg.has_max_elapsed = cc.has_max_elapsed = 0
cfg.epsilon = cc.epsilon = 1e-10
xg, rg = GpuOracle(A, mu, c).solve(cfg)
xc, rc = po.solve(A, mu, c, cc)
po.set_threads(2)
x2, r2 = po.solve(A, mu, c, cc)
po.set_threads(1)
for lab, x, r in (("gpu", xg, rg), ("cpu1", xc, rc), ("cpu2", x2, r2)):
    print(f"{lab}: status {r.status} ident {r.identification_steps} it {r.iterations} f {r.f_star:.12e} "
          f"kkt {r.kkt_residual:.1e} nact {int(np.sum(x <= cfg.tau + 1e-12))}")
