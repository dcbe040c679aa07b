"""Support size of the iterate over a solve (how small the faces get): python scripts/face_sizes.py C4"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import crra, make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
gamma = float(sys.argv[2]) if len(sys.argv) > 2 else None
A, mu, c = make_panel(name, seed=11)
if gamma:
    c = crra(gamma)
g = GpuOracle(A, mu, c)
cfg = preset("large")
cfg.has_max_elapsed = 0
sizes = []
g.solve(cfg, observer=lambda it, f, x: sizes.append((it, int(np.sum(x > cfg.tau + 1e-12)))))
print(name, "n", A.shape[1], "support per observer call:", sizes[:5], "...", sizes[-5:], "calls", len(sizes))
