"""Generate the committed golden fixtures under tests/golden/ (test
infrastructure). The reference (C++/Eigen) cannot be built in this image
(no Eigen), so the expected outputs come from the CPU restatement
in oracle/ — itself pinned by the reference's known-answer and relational
tests (tests/test_oracle_pins.py). The fixtures freeze those outputs on seeded
inputs so that (a) any later change to the restatement is caught on CPU
(tests/test_golden.py) and (b) the GPU path is checked against stored vectors
without running the oracle (tests/test_golden.py, -m gpu).

    python tests/golden/make_golden.py      # rewrites tests/golden/*.npz
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as po  # noqa: E402
from paper_2604_25378_b200.datagen import make_panel, random_simplex_point, random_tangents  # noqa: E402

OUT = Path(__file__).resolve().parent


def case(name, A, mu, c, seed, presets):
    T, n = A.shape
    o = po.CpuOracle(A, mu, c)
    x = random_simplex_point(n, seed)
    V = random_tangents(n, 4, seed)
    U = random_tangents(n, 4, seed + 1)
    cc = o.make_cache(x)
    f = o.value(cc)
    mom = np.array(o.moments(cc))
    g = o.gradient(cc)
    H = np.stack([o.hvp(cc, V[i]) for i in range(4)])
    T3 = np.stack([o.third_action(cc, U[i], V[i]) for i in range(4)])
    psi2 = o.hessian_diag_weights(cc)
    Ad = o.sample_direction(V[0])
    lm = o.line_model(cc, V[0], 0.05)
    d_direct, _ = o.yand_direction(cc, po.tangent_config("direct", lam=1e-6), 3)
    d_exact, _ = o.yand_direction(cc, po.tangent_config("pcg", lam=1e-4, krylov_tol=1e-12, krylov_maxit=200,
                                                         exact_trace=True), 3)
    sol = {}
    for p in presets:
        cfg = po.preset(p)
        cfg.has_max_elapsed = 0
        cfg.epsilon = 1e-10
        xs, rep = po.solve(A, mu, c, cfg)
        sol[f"x_{p}"] = xs
        sol[f"f_{p}"] = np.array([rep.f_star])
        sol[f"status_{p}"] = np.array([rep.status])
    np.savez_compressed(OUT / f"{name}.npz", A=A, mu=mu, c=c, x=x, V=V, U=U, f=np.array([f]), moments=mom, g=g,
                        H=H, T3=T3, psi2=psi2, Ad=Ad, line_model=lm, d_direct=d_direct, d_exact=d_exact, **sol)
    print(f"{name}: n={n} T={T} f={f:.6e} presets={presets}")


def main():
    po.set_threads(1)
    A, mu, c = make_panel("C1", seed=0)
    case("c1_small", A, mu, c, seed=11, presets=["small", "large"])
    A, mu, c = make_panel("C2", seed=0, kappa=100.0)
    A, mu = A[:400, :48].copy(), None  # a C2-generator slice (48 assets, 400 samples), re-centred below
    mu = A.mean(axis=0)
    A = A - mu
    case("c2_slice_k100", A, mu, c, seed=12, presets=["small"])


if __name__ == "__main__":
    main()
