"""The stress case's cluster-SPG endpoint, then the main loop from it on the GPU
and on the reference-exact CPU oracle (debugging aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

A, mu = rh.lcg_panel(12, 80, 32)
c = np.array([10.0, 1, 10, 1])
g = GpuOracle(A, mu, c)


def cfgs(**kw):
    out = []
    for mk in (preset, po.preset):
        cf = mk("large")
        cf.has_max_elapsed = 0
        cf.epsilon = 1e-10
        for k, v in kw.items():
            setattr(cf, k, v)
        out.append(cf)
    return out


cg, cc = cfgs(max_iter=0, stall_restarts=0)
x7, r7 = g.solve(cg)
x8, r8 = po.solve(A, mu, c, cc)
print("spg endpoints: gpu steps", r7.identification_steps, "cpu steps", r8.identification_steps,
      "dx %.3e" % float(np.max(np.abs(x7 - x8))))
np.set_printoptions(precision=17, linewidth=220)
print("gpu x7", x7)
print("cpu x8", x8)
cg, cc = cfgs(identification_pass=0 if isinstance(preset("large").identification_pass, int) else False)
for name, x0 in (("gpu-spg point", x7), ("cpu-spg point", x8)):
    xg, rg = g.solve(cg, x0=x0)
    xc, rc = po.solve(A, mu, c, cc, x0)
    print(name, "| gpu main loop:", rg.status, rg.iterations, rg.restarts, "kkt %.2e" % rg.kkt_residual,
          "| cpu main loop:", rc.status, rc.iterations, rc.restarts, "kkt %.2e" % rc.kkt_residual,
          "| dx %.3e" % float(np.max(np.abs(xg - xc))))
