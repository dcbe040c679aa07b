"""Run one op a few times on the C5 panel (for ncu captures): python scripts/prof_op.py hvp8 [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns  # noqa
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa

op = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = sys.argv[3] if len(sys.argv) > 3 else "C5"
spec = CONFIGS[cfg]
dev = torch.device("cuda", 0)
X = raw_returns(spec, 5000, device=dev)
mu_t = X.sum(0) / spec.T
X.sub_(mu_t)
T, n = spec.T, spec.n
ld = n if n < 512 else (n + 15) // 16 * 16  # the padded stride the host-upload path uses
if ld != n:
    Xp = torch.zeros((T, ld), dtype=X.dtype, device=dev)
    Xp[:, :n] = X
    X = Xp
gpu = GpuOracle(None, mu_t.cpu().numpy(), crra(spec.gamma), device_panel=(X.data_ptr(), ld, T, n))
xd = torch.from_numpy(random_simplex_point(n, 7)).to(dev)
Vd = torch.from_numpy(random_tangents(n, 8, 7)).to(dev)
out = torch.empty_like(Vd)
G = torch.empty((n, n), dtype=torch.float64, device=dev) if op == "gram" else None
gpu.make_cache_device(0, xd.data_ptr())
fn = {
    "hvp1": lambda: gpu.hvp_device(0, Vd.data_ptr(), 1, out.data_ptr()),
    "hvp4": lambda: gpu.hvp_device(0, Vd.data_ptr(), 4, out.data_ptr()),
    "hvp8": lambda: gpu.hvp_device(0, Vd.data_ptr(), 8, out.data_ptr()),
    "third8": lambda: gpu.third_action_device(0, Vd.data_ptr(), Vd.data_ptr(), 8, out.data_ptr()),
    "third": lambda: gpu.third_action_device(0, Vd.data_ptr(), Vd[1:].data_ptr(), 1, out.data_ptr()),
    "gram": lambda: gpu.weighted_gram_device(0, G.data_ptr()),
    "fgrad": lambda: gpu.make_cache_device(0, xd.data_ptr()),
}[op]
for _ in range(reps):
    fn()
gpu.synchronize()
print("ok", op)
