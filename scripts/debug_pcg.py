import os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import pyoracle as po
from paper_2604_25378_b200.datagen import make_panel
from paper_2604_25378_b200.gpu_oracle import GpuOracle, tangent_config
from tests import refhelpers as rh
A, mu, c = make_panel("C2", seed=4, kappa=10.0)
n = A.shape[1]
x = rh.simplex_point(n, 3, 1e-6)
cpu = po.CpuOracle(A, mu, c); cc = cpu.make_cache(x)
g = GpuOracle(A, mu, c)
for kw in (dict(lam=1e-4), dict(lam=1e-4, jacobi=True), dict(lam=0.0, krylov_tol=1e-12, krylov_maxit=200, exact_trace=True),
           dict(lam=1e-4, krylov_tol=1e-12, krylov_maxit=200, exact_trace=True), dict(lam=1e-4, probes=16), dict(lam=1e-4, probes=9)):
    gc = g.make_cache(x)
    dd, a = g.yand_direction(gc, tangent_config("pcg", **kw), 7)
    os.environ["MVSK_HOST_PCG"] = "1"
    gc = g.make_cache(x)
    dh, b = g.yand_direction(gc, tangent_config("pcg", **kw), 7)
    del os.environ["MVSK_HOST_PCG"]
    dc, cdg = cpu.yand_direction(cc, po.tangent_config("pcg", **kw), 7)
    print(kw, "iters", a.krylov_iters, b.krylov_iters, cdg.krylov_iters, "bd", a.pcg_breakdown, b.pcg_breakdown, cdg.pcg_breakdown,
          "dev-host %.2e dev-cpu %.2e host-cpu %.2e" % (np.max(np.abs(dd-dh)), np.max(np.abs(dd-dc)), np.max(np.abs(dh-dc))))
