"""Wide-row plans on a short panel (C4 by default): the default plan vs the
shared-memory-vector variant (MVSK_TUNE 6th field) for f+grad, 1-RHS HVP and
line sums; per-op time, GB/s and the max relative difference to the default
plan's result. python scripts/tune_vs.py [C4]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns  # noqa
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
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
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
gpu.set_stream(st.cuda_stream)
xd = torch.from_numpy(random_simplex_point(n, 7)).to(dev)
Vd = torch.from_numpy(random_tangents(n, 8, 7)).to(dev)
out = torch.zeros_like(Vd)
sums = torch.zeros(9, dtype=torch.float64, device=dev)
gpu.make_cache_device(0, xd.data_ptr())
alg = 8.0 * T * ld


def res_fgrad():
    gpu.make_cache_device(1, xd.data_ptr())
    gpu.synchronize()
    z, g, s = gpu.slot_pointers(1)
    return torch.frombuffer(bytearray(0), dtype=torch.float64) if False else None


FN = {
    "fgrad": (lambda: gpu.make_cache_device(1, xd.data_ptr()), None),
    "hvp1": (lambda: gpu.hvp_device(0, Vd.data_ptr(), 1, out.data_ptr()), lambda: out[0].clone()),
    "lines": (lambda: gpu.line_sums_device(0, Vd.data_ptr(), sums.data_ptr()), lambda: sums.clone()),
}


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


# MVSK_TUNE fields: Q, G, RG, S, OCC, VS
plans = ["", "8,1,2,2,0,0", "16,2,1,3,0,1", "16,2,1,2,0,1", "8,1,1,3,0,0"]
if len(sys.argv) > 2:
    plans = [""] + sys.argv[2:]
for op, (fn, get) in FN.items():
    ref = None
    for p in plans:
        if p:
            os.environ["MVSK_TUNE"] = p
        else:
            os.environ.pop("MVSK_TUNE", None)
        try:
            ms = timeit(fn)
            r = get() if get else None
        except Exception as e:  # noqa
            print(f"{cfg} {op} plan [{p}]: failed {e}", flush=True)
            continue
        if r is not None and ref is None:
            ref = r
        d = float((r - ref).abs().max() / ref.abs().max()) if r is not None else float("nan")
        print(f"{cfg} {op} plan [{p or 'default'}]: {ms * 1e3:.1f} us  {alg / ms / 1e6:.0f} GB/s  rel {d:.1e}",
              flush=True)
os.environ.pop("MVSK_TUNE", None)
