"""Warm-up solve, then one solve inside cudaProfilerStart/Stop (for
`ncu --profile-from-start off`): python scripts/one_solve_prof.py C4 [gamma|-] [large|small]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import crra, make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
gamma = float(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
mode = sys.argv[3] if len(sys.argv) > 3 else "large"
A, mu, c = make_panel(name, seed=11)
if gamma:
    c = crra(gamma)
g = GpuOracle(A, mu, c)
cfg = preset(mode)
cfg.has_max_elapsed = 0
g.solve(cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, rep = g.solve(cfg)
torch.cuda.profiler.stop()
print("ok", name, rep.iterations, rep.physical_passes, rep.wall_seconds)
