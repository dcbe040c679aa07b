"""Sweep streaming-kernel launch plans (MVSK_TUNE) on the C5 panel; prints ms and GB/s per op."""
import itertools
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns  # noqa
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["hvp1"]
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
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
gpu.set_stream(st.cuda_stream)
xd = torch.from_numpy(random_simplex_point(n, 7)).to(dev)
Vd = torch.from_numpy(random_tangents(n, 8, 7)).to(dev)
out = torch.empty_like(Vd)
sums = torch.empty(9, dtype=torch.float64, device=dev)
gpu.make_cache_device(0, xd.data_ptr())
alg = 8.0 * T * n
FN = {
    "hvp1": lambda: gpu.hvp_device(0, Vd.data_ptr(), 1, out.data_ptr()),
    "hvp2": lambda: gpu.hvp_device(0, Vd.data_ptr(), 2, out.data_ptr()),
    "hvp4": lambda: gpu.hvp_device(0, Vd.data_ptr(), 4, out.data_ptr()),
    "hvp8": lambda: gpu.hvp_device(0, Vd.data_ptr(), 8, out.data_ptr()),
    "third8": lambda: gpu.third_action_device(0, Vd.data_ptr(), Vd.data_ptr(), 8, out.data_ptr()),
    "fgrad": lambda: gpu.make_cache_device(1, xd.data_ptr()),
    "third": lambda: gpu.third_action_device(0, Vd.data_ptr(), Vd[1:].data_ptr(), 1, out.data_ptr()),
    "lines": lambda: gpu.line_sums_device(0, Vd.data_ptr(), sums.data_ptr()),
}


def timeit(fn, reps=10):
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


grid = [os.environ.get("MVSK_TUNE_GRID")] if os.environ.get("MVSK_TUNE_GRID") else None
for op in [o for o in ops if o in ("hvp8", "third8", "hvp4")]:
    for cl in ["dmma0", "dmma4,1", "dmma8,1", "dmma8,2", "dmma2,1", "0,0"]:
        if cl.startswith("dmma"):
            os.environ.pop("MVSK_NO_DMMA", None)
            os.environ["MVSK_TUNE_DMMA"] = os.environ.get("MVSK_TUNE_DMMA_FIX") or cl[4:]
        else:
            os.environ["MVSK_NO_DMMA"] = "1"
            os.environ["MVSK_TUNE_CLUSTER"] = cl
        try:
            ms = timeit(FN[op])
        except Exception as e:  # noqa
            print(f"{cfg} {op} cluster {cl}: failed {e}", flush=True)
            continue
        k = 8 if op.endswith("8") else 4
        print(f"{cfg} {op} cluster C,RG={cl}: {ms:.4f} ms  {alg / ms / 1e6:.0f} GB/s  {k * 1000 / ms:.0f} per s",
              flush=True)
    os.environ.pop("MVSK_TUNE_CLUSTER", None)
    os.environ.pop("MVSK_TUNE_DMMA", None)
    os.environ.pop("MVSK_NO_DMMA", None)
ops = [o for o in ops if o not in ("hvp8", "third8", "hvp4")]
for op in ops:
    os.environ.pop("MVSK_TUNE", None)
    base = timeit(FN[op])
    print(f"{cfg} {op} default: {base:.4f} ms  {alg / base / 1e6:.0f} GB/s", flush=True)
    if os.environ.get("TUNE_DEFAULT_ONLY"):
        continue
    for Q, G, RG, S, OCC in itertools.product([2, 4, 8], [1, 2, 4], [1, 2, 4], [2, 3, 4, 6], [1, 2]):
        if RG * Q > 8 and not (Q == 8 and RG == 2 and G == 1):
            continue
        os.environ["MVSK_TUNE"] = f"{Q},{G},{RG},{S},{OCC}"
        try:
            ms = timeit(FN[op])
        except Exception as e:  # noqa
            continue
        print(f"{cfg} {op} Q={Q} G={G} RG={RG} S={S} OCC={OCC}: {ms:.4f} ms  {alg / ms / 1e6:.0f} GB/s", flush=True)
os.environ.pop("MVSK_TUNE", None)
