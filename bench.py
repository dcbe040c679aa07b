#!/usr/bin/env python3
"""Benchmark: MVSK Hessian-vector products per second on the C5 configuration
(n=4096 assets, T=262144 samples, fp64; BASELINE.json configs[4]), row-sharded
over N GPUs of one node (one process per GPU, NCCL allreduce inside the C-ABI).

One step = one exact HVP  H v = A^T(psi''(z) o A v)/T over the whole panel
(oracle.hpp:92-101), inputs resident in HBM. The panel (8 GiB) is larger than
L2 (126 MB), so no L2 flush is needed between steps. Also reported on the same
line: fused f+grad, 8-RHS HVP, third action, line-search sums and the DMMA
weighted Gram; e2e through the host-pointer C-ABI; the CPU oracle baseline;
SM clocks sampled during the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MVSK HVPs/sec (exact fp64 Hessian-vector products, C5 n=4096 T=262144)"
UNIT = "HVP/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--seed", type=int, default=5000)
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary ops")
    ap.add_argument("--no-solve", action="store_true", help="skip the full-solve leg")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def hbm_peak():
    try:
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in Path(self.f.name).read_text().splitlines() if l.strip()]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                pass
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_hvp_rate(A_sample: np.ndarray, mu, c, T_full: int, threads: int, reps: int = 3):
    """CPU oracle HVP on a row sample: returns (HVP/s scaled to the full T, seconds per sampled HVP)."""
    from oracle import pyoracle as po
    po.set_threads(threads)
    Ts, n = A_sample.shape
    o = po.CpuOracle(A_sample, mu, c)
    x = np.full(n, 1.0 / n)
    cache = o.make_cache(x)
    v = np.random.default_rng(0).standard_normal(n)
    v -= v.mean()
    o.hvp(cache, v)  # warm-up (reference bench: 1 warm-up, lower median of reps)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        o.hvp(cache, v)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    t = ts[(len(ts) - 1) // 2]
    po.set_threads(1)
    return (Ts / T_full) / t, t


def solve_leg():
    """Full YAND solves (solver.hpp:195) through the C-ABI on BASELINE configs
    1-4 (config 2 at kappa 1 and 1000), GPU wall time (lower median of 3 after a warm-up; C4: 1 run) next to the
    CPU oracle restatement (1 thread, reference-faithful; C4 ~2.3 s since its
    face passes stream only the free columns). max_elapsed is disabled on both
    sides so both do the same work."""
    from oracle import pyoracle as po
    from paper_2604_25378_b200.datagen import crra, make_panel
    from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset
    out = []
    for name, kappa, mode, gamma, reps, cpu in (("C1", 1.0, "small", None, 3, True),
                                                ("C2", 1.0, "small", None, 3, True), ("C2", 1.0, "large", None, 3, True),
                                                ("C2", 1000.0, "large", None, 3, True),
                                                ("C3", 1.0, "large", 5.0, 3, True), ("C3", 1.0, "large", 20.0, 3, True),
                                                ("C4", 1.0, "large", None, 1, True)):
        A, mu, c = make_panel(name, seed=11, kappa=kappa)
        if gamma is not None:
            c = crra(gamma)
        g = GpuOracle(A, mu, c)
        cfg = preset(mode)
        cfg.has_max_elapsed = 0
        g.solve(cfg)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            x, rep = g.solve(cfg)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        row = {"config": name, "n": A.shape[1], "T": A.shape[0], "preset": mode, "gamma": gamma or 10.0, "kappa": kappa,
               "gpu_s": ts[(len(ts) - 1) // 2], "status": int(rep.status), "iterations": rep.iterations,
               "kkt": rep.kkt_residual, "physical_passes": int(rep.physical_passes),
               "logical_passes": int(rep.oracle_passes)}
        if cpu:
            cc = po.preset(mode)
            cc.has_max_elapsed = 0
            t0 = time.perf_counter()
            xc, rc = po.solve(A, mu, c, cc)
            row.update(cpu_s=time.perf_counter() - t0, cpu_status=int(rc.status), df=abs(rc.f_star - rep.f_star),
                       cpu_iterations=rc.iterations)
            # iteration counts are rounding-chaotic on both sides (the CPU oracle
            # with 2 threads moves them as much: scripts/iter_survey.py), so the
            # per-iteration times are the comparable pair
            row["gpu_ms_per_iter"] = 1e3 * row["gpu_s"] / max(1, rep.iterations)
            row["cpu_ms_per_iter"] = 1e3 * row["cpu_s"] / max(1, rc.iterations)
        if name == "C4":
            # BASELINE config 4's return-floor sweep: 5 floors between the
            # min-variance and max-mean means, c1 calibrated per floor
            t0 = time.perf_counter()
            sw = g.floor_sweep(cfg, nfloors=5)
            row["floor_sweep"] = {
                "wall_s": time.perf_counter() - t0, "solves": sw.total_solves, "m_mv": sw.m_mv, "m_max": sw.m_max,
                "points": [{k: p[k] for k in ("floor", "c1", "mean", "status", "solves")} for p in sw.points]}
        g.close()
        out.append(row)
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (the C++ restatement, since the
    Eigen-based reference cannot be compiled here) on all host cores, bounded sample."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import torch
    from paper_2604_25378_b200.datagen import CONFIGS, raw_returns
    spec = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    Ts = min(spec.T, 32768)
    R = raw_returns(spec, args.seed, rows=(0, Ts)).numpy()
    mu = R.sum(axis=0) / Ts
    A = R - mu
    from paper_2604_25378_b200.datagen import crra
    c = crra(spec.gamma)
    from oracle import pyoracle as po
    po.build()
    po.set_threads(cores)
    o = po.CpuOracle(A, mu, c)
    x = np.full(spec.n, 1.0 / spec.n)
    cache = o.make_cache(x)
    v = np.random.default_rng(0).standard_normal(spec.n)
    v -= v.mean()
    for _ in range(max(1, args.warmup)):
        o.hvp(cache, v)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.hvp(cache, v)
    dt = (time.perf_counter() - t0) / args.steps
    value = (Ts / spec.T) / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 * spec.T / Ts,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Student-t factor model, BASELINE.json config 5 shapes)",
        "config": {"workload": f"{args.config} HVP n={spec.n} T={spec.T}", "sample_rows": Ts},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"rows 0..{Ts} of the {args.config} panel, one HVP per step, scaled by T/{Ts}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns
    from paper_2604_25378_b200.gpu_oracle import GpuOracle, nccl_unique_id, shard_rows

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = CONFIGS[args.config]
    T, n = spec.T, spec.n
    row0, T_loc = shard_rows(T, ws, rank)

    # ---- panel shard in HBM (generated on device, centred with the global mean)
    X = raw_returns(spec, args.seed, rows=(row0, row0 + T_loc), device=dev)
    colsum = X.sum(dim=0)
    if ws > 1:
        dist.all_reduce(colsum)
    mu_t = colsum / T
    X.sub_(mu_t)
    mu = mu_t.cpu().numpy()
    c = crra(spec.gamma)
    nid = None
    if ws > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
    gpu = GpuOracle(None, mu, c, device=local, rank=rank, nranks=ws, row0=row0, T_global=T, nccl_id=nid,
                    device_panel=(X.data_ptr(), n, T_loc, n))
    # a dedicated stream: the context launches on it and the CUDA events time it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    gpu.set_stream(stream.cuda_stream)

    x = random_simplex_point(n, 7)
    V = random_tangents(n, 8, 7)
    xd = torch.from_numpy(x).to(dev)
    Vd = torch.from_numpy(V).to(dev)
    out = torch.empty_like(Vd)
    sums = torch.empty(9, dtype=torch.float64, device=dev)
    gpu.make_cache_device(0, xd.data_ptr())

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warm):
        for _ in range(warm):
            fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / steps)  # ms per call, max over ranks

    hvp1 = lambda: gpu.hvp_device(0, Vd.data_ptr(), 1, out.data_ptr())

    # ---- headline: single HVP, device-resident
    for _ in range(args.warmup):
        hvp1()
    barrier()
    clk = ClockSampler(local)
    time.sleep(0.3)
    l0 = gpu.launch_count()
    ms = timed(hvp1, args.steps, 0)
    # kernels the library enqueued in the timed region (counted inside the C-ABI:
    # one fused stream kernel per single-rank pass, + finish / allreduce otherwise)
    launches_total = gpu.launch_count() - l0
    clocks = clk.stop()
    value = 1000.0 / ms

    # per-op kernel time (events per call, on the launching stream): HBM roofline
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for a, b in evs:
        a.record(stream)
        hvp1()
        b.record(stream)
    barrier()
    per_launch_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in evs))
    alg_bytes = 8.0 * T_loc * n + 8.0 * T_loc + 16.0 * n  # one read of the shard + z + v/out
    peak, peak_kind = hbm_peak()
    achieved = alg_bytes / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    try:  # dram read+write per launch from the committed ncu --set full capture of this workload
        tr = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        if ws == 1 and args.config == "C5":
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read+write, profiles/ncu_traffic.json)",
                "algorithmic_bytes_per_launch": alg_bytes, "peak_kind": peak_kind,
                "note": "achieved = (8*T_local*n + 8*T_local + 16*n) B per HVP / mean per-call time of the "
                        "fused stream kernel (its cross-CTA reduction runs in the same cooperative launch), "
                        "CUDA events on the launching stream"}

    extra = {}
    if not args.no_extra:
        fgrad = lambda: gpu.make_cache_device(0, xd.data_ptr())
        extra["fgrad_ms"] = timed(fgrad, max(3, args.steps // 2), 2)
        extra["hvp8_ms"] = timed(lambda: gpu.hvp_device(0, Vd.data_ptr(), 8, out.data_ptr()), max(3, args.steps // 2), 1)
        extra["hvp8_per_s"] = 8000.0 / extra["hvp8_ms"]
        extra["third_ms"] = timed(lambda: gpu.third_action_device(0, Vd.data_ptr(), Vd[1:].data_ptr(), 1,
                                                                  out.data_ptr()), max(3, args.steps // 2), 1)
        extra["linesums_ms"] = timed(lambda: gpu.line_sums_device(0, Vd.data_ptr(), sums.data_ptr()),
                                     max(3, args.steps // 2), 1)
        for k in ("fgrad_ms", "third_ms", "linesums_ms"):
            extra[k.replace("_ms", "_GBps")] = alg_bytes / (extra[k] * 1e-3) / 1e9
        G = torch.empty((n, n), dtype=torch.float64, device=dev)
        gram_ms = timed(lambda: gpu.weighted_gram_device(0, G.data_ptr()), 1, 1)
        extra["gram_ms"] = gram_ms
        extra["gram_tflops"] = (T * n * (n + 1.0)) / (gram_ms * 1e-3) / 1e12
        try:  # fp64 tensor-pipe peak measured on this pool (profiles/r01_fp64_peak.json)
            pk = json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())["dmma_tflops"]
            extra["gram_roofline"] = {"bound": "tensor", "achieved": extra["gram_tflops"], "peak": pk,
                                      "unit": "TFLOP/s", "frac": extra["gram_tflops"] / pk,
                                      "flops_per_launch": T * n * (n + 1.0)}
        except Exception:
            pass
        # 8-RHS HVP / 8 third-action pairs: one HBM read of X (HBM roofline) and
        # 4*T*n*k (HVP) / 6*T*n*k (THIRD: two row dots per pair) flop on the
        # fp64 tensor pipe; both bounds reported, the larger fraction is binding
        extra["third8_ms"] = timed(lambda: gpu.third_action_device(0, Vd.data_ptr(), Vd.data_ptr(), 8,
                                                                   out.data_ptr()), max(3, args.steps // 2), 1)
        extra["hvp8_tflops"] = 4.0 * T_loc * n * 8 / (extra["hvp8_ms"] * 1e-3) / 1e12
        try:
            pk = json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())["dmma_tflops"]
        except Exception:
            pk = None
        for name, flop in (("hvp8", 4.0 * T_loc * n * 8), ("third8", 6.0 * T_loc * n * 8)):
            ms_k = extra[f"{name}_ms"]
            bytes_k = 8.0 * T_loc * n + 8.0 * T_loc + 24.0 * n * 8
            tf = flop / (ms_k * 1e-3) / 1e12
            gb = bytes_k / (ms_k * 1e-3) / 1e9
            extra[f"{name}_roofline"] = {
                "hbm": {"achieved": gb, "peak": peak, "unit": "GB/s", "frac": gb / peak},
                "tensor": {"achieved": tf, "peak": pk, "unit": "TFLOP/s", "frac": (tf / pk) if pk else None},
                "note": "warp-specialised DMMA kernel (stream_dmma_ws_kernel); 4-CTA clusters occupy 132 of "
                        "148 SMs, so the tensor ceiling on this launch is 132/148 of the peak"}
        del G

    # ---- e2e through the host-pointer C-ABI (pinned staging inside), per step: H2D v, D2H Hv
    from paper_2604_25378_b200.gpu_oracle import OracleCache
    cache0 = OracleCache(gpu, 0, float("nan"))
    vh = np.ascontiguousarray(V[0])
    for _ in range(args.warmup):
        gpu.hvp(cache0, vh)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        gpu.hvp(cache0, vh)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    e2e = {"value": 1.0 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
           "api": "mvsk_gpu_hvp (host pointers)"}

    # ---- CPU baseline (rank 0, N=1): oracle on a bounded row sample
    cpu_base = None
    if rank == 0 and ws == 1:
        Ts = min(T_loc, 32768)
        A_s = X[:Ts].cpu().numpy()
        rate, t_s = cpu_hvp_rate(A_s, mu, c, T, threads=1)
        cpu_base = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                    "sample": f"one HVP on rows 0..{Ts} of the same panel (2 reference passes), "
                              f"{t_s:.3f} s each, lower median of 3 after 1 warm-up, scaled by T/{Ts}"}

    # ---- YAND full-solve wall time (the metric's second half), rank 0 at N=1
    solves = None
    if rank == 0 and ws == 1 and not args.no_solve:
        solves = solve_leg()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 20-factor Student-t nu=5 panel, BASELINE.json config 5), generated on device",
            "config": {"workload": f"{args.config} single HVP, n={n} T={T}, rows sharded over {ws} GPU(s)",
                       "n": n, "T": T, "rows_per_gpu": T_loc, "l2": "panel 8 GiB > L2, no flush needed"},
            "roofline": roofline, "e2e": e2e, "gpu_launches": launches_total,
            "clocks": clocks, "ops": extra,
        }
        if cpu_base is not None:
            line["cpu_baseline"] = cpu_base
        if solves is not None:
            line["solve"] = solves
        print(json.dumps(line), flush=True)
    gpu.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
