"""One full solve of a BASELINE config (for ncu launch lists): python scripts/one_solve.py C4 [large]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
mode = sys.argv[2] if len(sys.argv) > 2 else "large"
A, mu, c = make_panel(name, seed=11)
g = GpuOracle(A, mu, c)
cfg = preset(mode)
cfg.has_max_elapsed = 0
x, rep = g.solve(cfg)
print("ok", name, rep.iterations, rep.physical_passes, rep.wall_seconds)
