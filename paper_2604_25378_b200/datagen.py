"""Seeded synthetic return panels for the BASELINE.json configurations.

The reference has no Student-t factor generator (its bench.hpp:25-77 draws
uniform or conditioned panels), so this module specifies the one
BASELINE.json describes. Everything is generated with torch so the same code
runs on the host (parity-test sizes, bit-reproducible from the seed) and on
the device (the 8 GiB C5 panel, where only the distribution matters).

Model, per config (daily returns, T periods x n assets):
    R[t, i] = drift_i + sum_k B[i, k] F[t, k] + idio_i * e[t, i]
    F[t, k] = fvol_k * s(t_nu)           (unit-variance Student-t shocks)
    e[t, i] = s(t_nu)
with s(t_nu) = t_nu * sqrt((nu - 2) / nu). C3 additionally skews the factors
with a sign-biased lognormal multiplier: negative factor shocks are scaled by
exp(0.5 N - 0.125) (mean-one lognormal), positive ones are not, which gives
negatively skewed factor returns. The panel is then centred (panel.hpp:32-44):
X = R - 1 mu^T, mu = column means. Column rescaling for C2: s_j = kappa^(j/(n-1)).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class PanelSpec:
    name: str
    n: int
    T: int
    factors: int
    nu: int
    fvol_lo: float
    fvol_hi: float
    idio_lo: float
    idio_hi: float
    drift_hi: float = 5e-4
    skew: bool = False
    kappa: float = 1.0
    gamma: float = 10.0


CONFIGS = {
    "C1": PanelSpec("C1", 20, 500, 3, 5, 0.01, 0.01, 0.005, 0.02),
    "C2": PanelSpec("C2", 100, 1000, 3, 5, 0.01, 0.01, 0.005, 0.02),
    "C3": PanelSpec("C3", 800, 2500, 10, 4, 0.01, 0.03, 0.01, 0.03, skew=True, gamma=5.0),
    "C4": PanelSpec("C4", 5000, 5000, 20, 5, 0.01, 0.01, 0.005, 0.03),
    "C5": PanelSpec("C5", 4096, 262144, 20, 5, 0.01, 0.01, 0.005, 0.03),
}


def crra(gamma: float) -> np.ndarray:
    """panel.hpp:76-87"""
    g = float(gamma)
    return np.array([1.0, g / 2.0, g * (g + 1.0) / 6.0, g * (g + 1.0) * (g + 2.0) / 24.0])


def _student(gen: torch.Generator, shape, nu: int, device, dtype=torch.float64) -> torch.Tensor:
    z = torch.randn(shape, generator=gen, device=device, dtype=dtype)
    chi2 = torch.zeros(shape, device=device, dtype=dtype)
    for _ in range(nu):
        chi2.add_(torch.randn(shape, generator=gen, device=device, dtype=dtype).square_())
    return z / torch.sqrt(chi2 / nu) * np.sqrt((nu - 2.0) / nu)


def _asset_params(spec: PanelSpec, seed: int):
    """Loadings, idiosyncratic vols, drifts and factor vols (host, float64)."""
    g = torch.Generator(device="cpu").manual_seed(seed * 7919 + 17)
    B = torch.randn((spec.n, spec.factors), generator=g, dtype=torch.float64) * 0.3
    B[:, 0] += 1.0  # loadings N(1, 0.3^2) on factor 1, N(0, 0.3^2) on the rest
    idio = spec.idio_lo + (spec.idio_hi - spec.idio_lo) * torch.rand(spec.n, generator=g, dtype=torch.float64)
    drift = spec.drift_hi * torch.rand(spec.n, generator=g, dtype=torch.float64)
    fvol = spec.fvol_lo + (spec.fvol_hi - spec.fvol_lo) * torch.rand(spec.factors, generator=g, dtype=torch.float64)
    return B, idio, drift, fvol


def raw_returns(spec: PanelSpec, seed: int, rows: tuple[int, int] | None = None, device="cpu",
                chunk: int = 16384, kappa: float | None = None) -> torch.Tensor:
    """Raw returns R[rows] (T_rows x n). Rows are generated in fixed chunks
    seeded by (seed, chunk index), so any row block (e.g. one rank's shard) is
    reproducible on its own."""
    lo, hi = rows if rows is not None else (0, spec.T)
    B, idio, drift, fvol = (t.to(device) for t in _asset_params(spec, seed))
    kap = spec.kappa if kappa is None else kappa
    scale = None
    if kap != 1.0:
        j = torch.arange(spec.n, device=device, dtype=torch.float64)
        scale = kap ** (j / max(spec.n - 1, 1))
    out = torch.empty((hi - lo, spec.n), device=device, dtype=torch.float64)
    c0 = lo // chunk
    c1 = (hi + chunk - 1) // chunk
    for c in range(c0, c1):
        r_lo, r_hi = c * chunk, min((c + 1) * chunk, spec.T)
        g = torch.Generator(device=device).manual_seed(int(seed) * 1_000_003 + c)
        m = r_hi - r_lo
        F = _student(g, (m, spec.factors), spec.nu, device) * fvol
        if spec.skew:
            L = torch.exp(0.5 * torch.randn((m, spec.factors), generator=g, device=device, dtype=torch.float64) - 0.125)
            F = torch.where(F < 0, F * L, F)
        E = _student(g, (m, spec.n), spec.nu, device)
        R = drift + F @ B.T + E * idio
        if scale is not None:
            R = R * scale
        a, b = max(lo, r_lo), min(hi, r_hi)
        out[a - lo:b - lo] = R[a - r_lo:b - r_lo]
    return out


def make_panel(spec: PanelSpec | str, seed: int = 0, kappa: float | None = None):
    """Host panel: (A, mu, c) as numpy float64 — centred X, column means, CRRA coefficients."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    R = raw_returns(spec, seed, kappa=kappa).numpy()
    mu = R.sum(axis=0) / R.shape[0]
    return R - mu[None, :], mu, crra(spec.gamma)


def random_simplex_point(n: int, seed: int) -> np.ndarray:
    """Random interior simplex point: normalised exponentials."""
    rng = np.random.default_rng(seed)
    e = rng.exponential(size=n)
    return e / e.sum()


def random_tangents(n: int, k: int, seed: int) -> np.ndarray:
    """k tangent directions v ~ N(0, I) projected to sum(v) = 0."""
    rng = np.random.default_rng(seed + 99991)
    V = rng.standard_normal((k, n))
    return V - V.mean(axis=1, keepdims=True)
