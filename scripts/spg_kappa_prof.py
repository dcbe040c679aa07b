import sys
sys.path.insert(0, '.')
from paper_2604_25378_b200.datagen import make_panel
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset
A, mu, c = make_panel("C2", seed=11, kappa=1000.0)
cfg = preset("large"); cfg.has_max_elapsed = 0
g = GpuOracle(A, mu, c)
x, r = g.solve(cfg)
print("ok", r.identification_steps)
