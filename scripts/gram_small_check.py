"""weighted_gram on small panels vs numpy (debugging aid for the one-cluster Gram)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_25378_b200.gpu_oracle import GpuOracle  # noqa: E402
from tests import refhelpers as rh  # noqa: E402

for n, T in [(20, 500), (24, 64), (64, 500), (64, 2000), (100, 1000), (128, 900), (8, 100), (16, 100)]:
    rng = np.random.default_rng(n + T)
    A = rng.uniform(-0.1, 0.4, (T, n))
    A -= A.mean(axis=0)
    c = rh.crra(10.0)
    g = GpuOracle(A, np.zeros(n), c)
    x = rh.simplex_point(n, 1)
    gc = g.make_cache(x)
    z = A @ x
    psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
    ref = (A * psi2[:, None]).T @ A / T
    G = g.weighted_gram(gc)
    err = np.abs(G - ref)
    bad = np.argwhere(err > 1e-12 * np.abs(ref).max())
    print(n, T, "max rel err %.2e" % (err.max() / np.abs(ref).max()), "bad", len(bad), bad[:6].tolist(),
          "ratio diag", np.round((np.diag(G) / np.diag(ref))[:8], 3).tolist(), flush=True)
    g.close()
