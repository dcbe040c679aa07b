"""Latency of single passes on a narrow panel (a compact C4 face: T=5000, n=64):
python scripts/small_pass_bench.py [T] [n]. Sweeps MVSK_TUNE plans for k=1 HVP."""
import itertools
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
rng = np.random.default_rng(0)
A = rng.standard_normal((T, n)) * 0.01
mu = A.mean(0)
A -= mu
g = GpuOracle(A, mu, [1.0, 5.0, 18.3, 55.0])
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
g.set_stream(st.cuda_stream)
x = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
V = torch.randn(8, n, dtype=torch.float64, device=dev)
out = torch.empty_like(V)
g.make_cache_device(0, x.data_ptr())


def t(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for k in (1, 8):
    print(f"T={T} n={n} hvp k={k}: {t(lambda: g.hvp_device(0, V.data_ptr(), k, out.data_ptr())):.2f} us", flush=True)
print(f"fgrad: {t(lambda: g.make_cache_device(1, x.data_ptr())):.2f} us", flush=True)
best = []
for Q, G, RG, S, OCC in itertools.product([1, 2, 4, 8], [1, 2, 4, 8, 16], [1, 2, 4], [2, 3], [1]):
    os.environ["MVSK_TUNE"] = f"{Q},{G},{RG},{S},{OCC}"
    try:
        us = t(lambda: g.hvp_device(0, V.data_ptr(), 1, out.data_ptr()), 100)
    except Exception:
        continue
    best.append((us, Q, G, RG, S, OCC))
os.environ.pop("MVSK_TUNE")
best.sort()
for b in best[:3]:
    print("k=1 tune %.2f us  Q=%d G=%d RG=%d S=%d OCC=%d" % b)
