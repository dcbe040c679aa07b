"""A/B of the Gram-PCG direction (gram_pcg.cu) against the matrix-free device
PCG (MVSK_NO_GRAM_PCG) and the CPU reference restatement: directions,
Krylov counts and solve results/times on BASELINE configs. Each variant runs in
its own process (the switch is read once)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r'''
import sys, json, time, numpy as np
sys.path.insert(0, %r)
from paper_2604_25378_b200.datagen import make_panel, crra, random_simplex_point
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset, tangent_config
from oracle import pyoracle as po
out = {}
for name, kappa, gamma in (("C2", 1.0, None), ("C2", 1000.0, None), ("C3", 1.0, 5.0), ("C3", 1.0, 20.0), ("C4", 1.0, None)):
    A, mu, c = make_panel(name, seed=11, kappa=kappa)
    if gamma: c = crra(gamma)
    key = f"{name}_k{kappa:g}_g{gamma or 10:g}"
    g = GpuOracle(A, mu, c)
    cfg = preset("large"); cfg.has_max_elapsed = 0
    g.solve(cfg)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); x, r = g.solve(cfg); ts.append(time.perf_counter() - t0)
    cfg2 = preset("large"); cfg2.has_max_elapsed = 0; cfg2.epsilon = 1e-10
    x2, r2 = g.solve(cfg2)
    cc = po.preset("large"); cc.has_max_elapsed = 0; cc.epsilon = 1e-10
    xc, rc = po.solve(A, mu, c, cc)
    # one direction on a narrow face: the first 40 assets of the panel
    n = A.shape[1]
    idx = np.arange(min(n, 40))
    x0 = np.full(n, 1e-8); x0[idx] = (1 - 1e-8 * (n - len(idx))) / len(idx)
    g.set_face(idx, 1e-8)
    gc = g.make_cache(x0[idx])
    d, dg = g.yand_direction(gc, tangent_config("pcg", lam=1e-4), 5)
    g.set_face()
    out[key] = dict(solve_ms=sorted(ts)[1] * 1e3, it=r.iterations, status=r.status, f=r.f_star,
                    dx_ref_1e10=float(np.abs(x2 - xc).max()), st_ref=[r2.status, rc.status],
                    d=d.tolist(), kry=dg.krylov_iters)
    g.close()
print(json.dumps(out))
''' % str(ROOT)
res = {}
for tag, env in (("gram", {}), ("matfree", {"MVSK_NO_GRAM_PCG": "1"})):
    r = subprocess.run([sys.executable, "-c", CODE], env={**os.environ, **env}, capture_output=True, text=True)
    if r.returncode != 0:
        print(tag, "FAILED", r.stderr[-3000:])
        continue
    res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
for key in res.get("gram", {}):
    a, b = res["gram"][key], res.get("matfree", {}).get(key, {})
    dd = max(abs(u - v) for u, v in zip(a["d"], b["d"])) / max(abs(v) for v in b["d"]) if b else float("nan")
    print(f"{key}: solve {a['solve_ms']:.2f} ms (matfree {b.get('solve_ms', float('nan')):.2f}) it {a['it']}/{b.get('it')} "
          f"dx_ref(1e-10) {a['dx_ref_1e10']:.1e}/{b.get('dx_ref_1e10', float('nan')):.1e} status {a['st_ref']} "
          f"dir rel {dd:.1e} krylov {a['kry']}/{b.get('kry')}")
