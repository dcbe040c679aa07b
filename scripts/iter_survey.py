"""Iteration counts of GPU vs CPU-oracle solves over seeds (trajectory
sensitivity check): python scripts/iter_survey.py C1 small 10"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.datagen import make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
mode = sys.argv[2] if len(sys.argv) > 2 else "small"
nseeds = int(sys.argv[3]) if len(sys.argv) > 3 else 10
gi, ci = [], []
for seed in range(nseeds):
    A, mu, c = make_panel(name, seed=seed)
    cfg, cc = preset(mode), po.preset(mode)
    cfg.has_max_elapsed = cc.has_max_elapsed = 0
    g = GpuOracle(A, mu, c)
    xg, rg = g.solve(cfg)
    g.close()
    xc, rc = po.solve(A, mu, c, cc)
    x2 = None
    po.set_threads(2)
    try:
        x2, r2 = po.solve(A, mu, c, cc)
    finally:
        po.set_threads(1)
    gi.append(rg.iterations)
    ci.append(rc.iterations)
    print(f"seed {seed}: gpu {rg.iterations:3d} it (status {rg.status}), cpu {rc.iterations:3d} it, cpu-2thr {r2.iterations:3d} it,"
          f" |dx| {np.max(np.abs(xg - xc)):.1e}, df {abs(rg.f_star - rc.f_star):.1e}", flush=True)
print("mean gpu", np.mean(gi), "mean cpu", np.mean(ci))
