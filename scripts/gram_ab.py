"""A/B of the weighted-Gram warp layouts (MVSK_GRAM_VAR) on the C5 panel:
python scripts/gram_ab.py [C5] [variants...]"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, raw_returns  # noqa
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
variants = sys.argv[2:] or ["0", "1", "2"]
spec = CONFIGS[cfg]
dev = torch.device("cuda", 0)
X = raw_returns(spec, 5000, device=dev)
mu_t = X.sum(0) / spec.T
X.sub_(mu_t)
T, n = spec.T, spec.n
ld = n if n < 512 else (n + 15) // 16 * 16
if ld != n:
    Xp = torch.zeros((T, ld), dtype=X.dtype, device=dev)
    Xp[:, :n] = X
    X = Xp
gpu = GpuOracle(None, mu_t.cpu().numpy(), crra(spec.gamma), device_panel=(X.data_ptr(), ld, T, n))
xd = torch.from_numpy(random_simplex_point(n, 7)).to(dev)
gpu.make_cache_device(0, xd.data_ptr())
ref = None
for v in variants:
    os.environ["MVSK_GRAM_VAR"] = v
    G = torch.empty((n, n), dtype=torch.float64, device=dev)
    gpu.weighted_gram_device(0, G.data_ptr())
    gpu.synchronize()
    s = gpu.stream_handle() if hasattr(gpu, "stream_handle") else None
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        gpu.weighted_gram_device(0, G.data_ptr())
        gpu.synchronize()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[1]
    err = 0.0 if ref is None else float(((G - ref).abs().max() / ref.abs().max()).item())
    if ref is None:
        ref = G.clone()
    print(f"{cfg} var {v}: {ms:.2f} ms  {T * n * (n + 1.0) / (ms * 1e-3) / 1e12:.2f} TFLOP/s  relerr vs var {variants[0]}: {err:.1e}", flush=True)
