"""Replays test_stress_profiles_direct_and_pcg's sequence for one profile and
prints every solve's outcome (debugging aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset, tangent_config  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

c = np.array([float(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "10,1,10,1").split(",")])
skip = set(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] else set()
dsel = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 and sys.argv[3] else [0, 1, 2]
presets = sys.argv[4].split(",") if len(sys.argv) > 4 else ["small", "large"]
for seed, (n, T) in enumerate([(6, 40), (12, 80), (25, 200)]):
    if seed in skip:
        continue
    A, mu = rh.lcg_panel(n, T, seed + 31)
    cpu, gpu = po.CpuOracle(A, mu, c), GpuOracle(A, mu, c)
    x = rh.simplex_point(n, seed + 3, 1e-6)
    cc, gc = cpu.make_cache(x), gpu.make_cache(x)
    for k, (mode, lam) in enumerate((("direct", 0.0), ("direct", 1e-6), ("pcg", 1e-4))):
        if k not in dsel:
            continue
        dc, ddc = cpu.yand_direction(cc, po.tangent_config(mode, lam=lam), seed)
        dg, ddg = gpu.yand_direction(gc, tangent_config(mode, lam=lam), seed)
        print(n, mode, lam, "dir dx", float(np.max(np.abs(dg - dc))), ddg.krylov_iters, ddc.krylov_iters)
    for pre in presets:
        cfg_c, cfg_g = po.preset(pre), preset(pre)
        for cfg in (cfg_c, cfg_g):
            cfg.has_max_elapsed = 0
            cfg.epsilon = 1e-10
        xg, rg = gpu.solve(cfg_g)
        xc, rc = po.solve(A, mu, c, cfg_c)
        print(n, pre, "gpu", rg.status, rg.iterations, rg.face_events, rg.restarts, "cpu", rc.status, rc.iterations,
              rc.face_events, rc.restarts, "dx", float(np.max(np.abs(xg - xc))), "kkt", rg.kkt_residual, rc.kkt_residual,
              "f", rg.f_star, rc.f_star, "ident", rg.identification_steps, rc.identification_steps, flush=True)
    gpu.close()
