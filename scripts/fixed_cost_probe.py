"""Fixed cost of a wide-row pass: the same n = 5000 panel truncated to T rows (the streaming part scales
with T, the launch / prologue / grid barrier / cross-CTA reduction do not). python scripts/fixed_cost_probe.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns  # noqa
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa

spec = CONFIGS["C4"]
dev = torch.device("cuda", 0)
X = raw_returns(spec, 5000, device=dev)
mu_t = X.sum(0) / spec.T
X.sub_(mu_t)
n = spec.n
ld = (n + 15) // 16 * 16
Xp = torch.zeros((spec.T, ld), dtype=X.dtype, device=dev)
Xp[:, :n] = X
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
xd = torch.from_numpy(random_simplex_point(n, 7)).to(dev)
Vd = torch.from_numpy(random_tangents(n, 8, 7)).to(dev)
out = torch.zeros_like(Vd)
sums = torch.zeros(9, dtype=torch.float64, device=dev)
for T in (148, 296, 592, 1184, 2368, 5000):
    gpu = GpuOracle(None, mu_t.cpu().numpy(), crra(spec.gamma), device_panel=(Xp.data_ptr(), ld, T, n))
    gpu.set_stream(st.cuda_stream)
    gpu.make_cache_device(0, xd.data_ptr())
    line = [f"T={T:5d} rows/CTA={T / 148:5.1f}:"]
    for name, fn in (("fgrad", lambda: gpu.make_cache_device(1, xd.data_ptr())),
                     ("hvp1", lambda: gpu.hvp_device(0, Vd.data_ptr(), 1, out.data_ptr())),
                     ("lines", lambda: gpu.line_sums_device(0, Vd.data_ptr(), sums.data_ptr()))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(50):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        line.append(f"{name} {a.elapsed_time(b) / 50 * 1e3:6.1f} us |")
    print(" ".join(line), flush=True)
    gpu.close()
