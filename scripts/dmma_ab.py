"""A/B timing of the multi-RHS tensor-core passes: warp-specialised kernel
(ws, the default) vs v1 (MVSK_DMMA_V1=1), plus a relative comparison of the
results. python scripts/dmma_ab.py C5 hvp8,third8,hvp4 ws,v1
(another build of the library: MVSK_B200_LIB=<path> python scripts/dmma_ab.py C5 hvp8 ws)"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns  # noqa
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["hvp8", "third8"]
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["ws", "v1"]
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
Ud = torch.from_numpy(random_tangents(n, 8, 8)).to(dev)
out = torch.zeros_like(Vd)
gpu.make_cache_device(0, xd.data_ptr())
FN = {
    "hvp4": (4, lambda: gpu.hvp_device(0, Vd.data_ptr(), 4, out.data_ptr())),
    "hvp8": (8, lambda: gpu.hvp_device(0, Vd.data_ptr(), 8, out.data_ptr())),
    "third4": (4, lambda: gpu.third_action_device(0, Ud.data_ptr(), Vd.data_ptr(), 4, out.data_ptr())),
    "third8": (8, lambda: gpu.third_action_device(0, Ud.data_ptr(), Vd.data_ptr(), 8, out.data_ptr())),
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


alg = 8.0 * T * ld
for op in ops:
    k, fn = FN[op]
    res = {}
    for var in variants:
        os.environ.pop("MVSK_DMMA_V1", None)
        if var == "v1":
            os.environ["MVSK_DMMA_V1"] = "1"
        out.zero_()
        fn()
        torch.cuda.synchronize()
        res[var] = out[:k].clone()
        ms = timeit(fn)
        print(f"{cfg} {op} {var}: {ms:.4f} ms  {alg / ms / 1e6:.0f} GB/s  {k * 1000 / ms:.0f} per s", flush=True)
    ref = res[variants[-1]]
    for var in variants[:-1]:
        d = (res[var] - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
        print(f"{cfg} {op} {var} vs {variants[-1]}: max rel diff {d:.3e}", flush=True)
