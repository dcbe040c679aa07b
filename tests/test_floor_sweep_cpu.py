"""Host logic of the return-floor sweep (BASELINE config 4) on the CPU oracle:
each calibrated optimum lands within the mean tolerance of its floor, and the
calibrated c1 and means increase with the floor."""
import numpy as np

from oracle import pyoracle as po
from tests import refhelpers as rh


def test_floor_sweep_mirror_on_cpu_oracle():
    A, mu = rh.lcg_panel(8, 120, 21)
    mu = mu + np.linspace(0.0, 0.02, 8)  # spread the asset means
    c = rh.crra(10.0)
    cfg = po.preset("small")
    cfg.has_max_elapsed = 0

    def solve_fn(coeffs, x0):
        return po.solve(A, mu, coeffs, cfg, x0)[0]

    out = rh.floor_sweep_ref(solve_fn, mu, c, nfloors=3, mean_tol=1e-3, max_solves=24)
    span = out["m_max"] - out["m_mv"]
    assert span > 0
    c1s = [b["c1"] for b in out["best"]]
    means = [b["mean"] for b in out["best"]]
    for r, m in zip(out["floors"], means):
        assert abs(m - r) <= 1e-3 * span + 1e-15, (r, m)
    assert all(np.diff(c1s) > 0) and all(np.diff(means) > 0)
    assert out["floors"][0] > out["m_mv"] and out["floors"][-1] < out["m_max"]
