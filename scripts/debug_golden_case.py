"""Diagnose a golden-fixture solve mismatch on the GPU: run the fixture's
preset solves (epsilon 1e-10) under each A/B switch in a fresh process and
print status / iterations / kkt / |dx| against the reference's stored x."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
name = sys.argv[1] if len(sys.argv) > 1 else "lcg_n9_T60"
CODE = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset
g = dict(np.load(%r))
out = {}
for p in ("small", "large"):
    if f"x_{p}" not in g: continue
    cfg = preset(p); cfg.has_max_elapsed = 0; cfg.epsilon = 1e-10
    traj = []
    gpu = GpuOracle(g["A"], g["mu"], g["c"])
    x, r = gpu.solve(cfg, observer=lambda it, f, xx: traj.append((it, f)))
    out[p] = dict(status=r.status, it=r.iterations, kkt=r.kkt_residual, dx=float(np.abs(x - g[f"x_{p}"]).max()),
                  ref_status=int(g[f"status_{p}"][0]), faces=r.face_events, restarts=r.restarts,
                  ident=r.identification_steps, tail=[(i, f) for i, f in traj[-6:]])
print(json.dumps(out))
''' % (str(ROOT), str(ROOT / "tests" / "golden" / f"{name}.npz"))
for env in ({}, {"MVSK_NO_GRAPHS": "1"}, {"MVSK_NO_SPG_CLUSTER": "1"}, {"MVSK_NO_CCG": "1"}, {"MVSK_HOST_PCG": "1"},
            {"MVSK_NO_FUSED_FINISH": "1"}, {"MVSK_NO_CG_GRAPH": "1", "MVSK_NO_DIR_GRAPH": "1"}):
    r = subprocess.run([sys.executable, "-c", CODE], env={**os.environ, **env}, capture_output=True, text=True)
    print(env, r.stdout.strip() or r.stderr[-800:], flush=True)
