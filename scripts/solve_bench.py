"""YAND full-solve wall time, GPU driver vs the CPU oracle restatement, on the
BASELINE.json configurations 1-4 (seeded synthetic panels). max_elapsed is
disabled on both sides so the work is comparable; CPU solves are skipped above
--cpu-max-n to keep the run bounded.

  python scripts/solve_bench.py [--configs C1,C2,C3,C4] [--cpu-max-n 800] [--reps 3]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_25378_b200.datagen import CONFIGS, crra, make_panel  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402


def cases(names):
    out = []
    for name in names:
        if name == "C1":
            out.append(("C1", 1.0, "small", None))
        elif name == "C2":
            for k in (1.0, 10.0, 100.0, 1000.0):
                out.append(("C2", k, "small", None))
                out.append(("C2", k, "large", None))
        elif name == "C3":
            for g in (5.0, 20.0):
                out.append(("C3", 1.0, "large", g))
        elif name == "C4":
            out.append(("C4", 1.0, "large", None))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3")
    ap.add_argument("--cpu-max-n", type=int, default=800)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from oracle import pyoracle as po
    rows = []
    for name, kappa, mode, gamma in cases(args.configs.split(",")):
        A, mu, c = make_panel(name, seed=11, kappa=kappa)
        if gamma is not None:
            c = crra(gamma)
        T, n = A.shape
        gpu = GpuOracle(A, mu, c)
        cfg = preset(mode)
        cfg.has_max_elapsed = 0
        gpu.solve(cfg)  # warm-up (reference bench: 1 warm-up, lower median of reps)
        ts, rep = [], None
        for _ in range(args.reps):
            t0 = time.perf_counter()
            x, rep = gpu.solve(cfg)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        row = {"config": name, "kappa": kappa, "gamma": gamma or CONFIGS[name].gamma, "preset": mode, "n": n, "T": T,
               "gpu_s": ts[(len(ts) - 1) // 2], "gpu_status": int(rep.status), "gpu_iters": rep.iterations,
               "gpu_kkt": rep.kkt_residual, "logical_passes": int(rep.oracle_passes),
               "physical_passes": int(rep.physical_passes), "f": rep.f_star}
        if n <= args.cpu_max_n:
            cc = po.preset(mode)
            cc.has_max_elapsed = 0
            t0 = time.perf_counter()
            xc, rc = po.solve(A, mu, c, cc)
            row.update(cpu_s=time.perf_counter() - t0, cpu_status=int(rc.status), cpu_iters=rc.iterations,
                       cpu_passes=int(rc.oracle_passes), df=abs(rc.f_star - rep.f_star),
                       dx=float(np.max(np.abs(xc - x))))
        rows.append(row)
        print(json.dumps(row), flush=True)
    gpu = None


if __name__ == "__main__":
    main()
