"""Independent test references, restating the reference suite's helpers
(/root/reference/proj/tests/helpers.hpp, test_oracle.cpp:13-25,
test_solver.cpp:15-28) in plain numpy / Python loops — no shared code with
either the oracle restatement or the CUDA product."""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def _lcg_stream(state: int):
    s = state
    while True:
        s = (s * 6364136223846793005 + 1442695040888963407) & M64
        yield (s >> 11) / 9007199254740992.0


def center(R: np.ndarray):
    """center_panel (panel.hpp:32-44): mu = column means, A = R - 1 mu^T."""
    mu = R.mean(axis=0)
    return R - mu[None, :], mu


def lcg_panel_raw(n: int, T: int, seed: int) -> np.ndarray:
    """helpers.hpp:119-129: LCG U[-0.1, 0.4) panel (raw returns R, T x n)."""
    g = _lcg_stream(seed)
    R = np.empty((T, n))
    for t in range(T):
        for i in range(n):
            R[t, i] = -0.1 + 0.5 * next(g)
    return R


def lcg_panel(n: int, T: int, seed: int):
    """Returns (A, mu) of the centred lcg panel. Centring follows
    center_panel's mean (sum / T) exactly."""
    R = lcg_panel_raw(n, T, seed)
    mu = R.sum(axis=0) / T
    return R - mu[None, :], mu


def simplex_point(n: int, seed: int, tau: float = 0.0) -> np.ndarray:
    """helpers.hpp:131-146"""
    g = _lcg_stream((seed * 2654435761 + 1) & M64)
    x = np.array([0.05 + next(g) for _ in range(n)])
    scale = (1.0 - n * tau) / x.sum()
    return tau + x * scale


def ref_value(A, mu, c, x) -> float:
    """helpers.hpp:23-36 plain-loop objective."""
    z = A @ x
    z2 = z * z
    acc = float(np.sum(c[1] * z2 - c[2] * z2 * z + c[3] * z2 * z2))
    return -c[0] * float(mu @ x) + acc / A.shape[0]


def loop_gradient(A, mu, c, x) -> np.ndarray:
    """test_oracle.cpp:13-25"""
    T = A.shape[0]
    z = A @ x
    w = (2 * c[1] * z - 3 * c[2] * z * z + 4 * c[3] * z ** 3) / T
    return -c[0] * mu + A.T @ w


def ref_hvp(A, c, x, v) -> np.ndarray:
    T = A.shape[0]
    z = A @ x
    return A.T @ ((2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z) * (A @ v) / T)


def ref_third(A, c, x, u, v) -> np.ndarray:
    T = A.shape[0]
    z = A @ x
    return A.T @ ((-6 * c[2] + 24 * c[3] * z) * (A @ u) * (A @ v) / T)


def fd_gradient(f, x, h):
    g = np.empty(x.size)
    for i in range(x.size):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


def fd_directional(field, x, u, h):
    return (field(x + h * u) - field(x - h * u)) / (2 * h)


def grid_line_min(phi, cap, points=100000):
    a = cap * np.arange(0, points + 1) / points
    v = phi(a)
    k = int(np.argmin(v))
    return a[k], v[k]


def is_valid_projection(v, y, tau, mass, tol=1e-9) -> bool:
    """helpers.hpp:73-95"""
    if np.any(y < tau - tol):
        return False
    if abs(y.sum() - mass) > tol * max(1.0, abs(mass)):
        return False
    theta = None
    for i in range(y.size):
        if y[i] > tau + tol:
            if theta is None:
                theta = v[i] - y[i]
            elif abs(v[i] - y[i] - theta) > tol:
                return False
    if theta is not None:
        for i in range(y.size):
            if y[i] <= tau + tol and v[i] - tau > theta + tol:
                return False
    return True


def mv_two_asset_optimum(A, mu, c1, c2, tau):
    """helpers.hpp:98-116"""
    T = A.shape[0]
    d = A[:, 0] - A[:, 1]
    p = float(d @ d) / T
    q = float(A[:, 1] @ d) / T
    r0 = float(A[:, 1] @ A[:, 1]) / T
    dmu = mu[0] - mu[1]
    w = (c1 * dmu - 2 * c2 * q) / (2 * c2 * p)
    w = min(max(w, tau), 1 - tau)
    f = -c1 * (mu[1] + dmu * w) + c2 * (r0 + 2 * q * w + p * w * w)
    return w, f


def dominated_panel(T: int):
    """test_solver.cpp:15-28: asset 2 is dominated and must be pinned."""
    g = _lcg_stream(42)
    R = np.empty((T, 3))
    for t in range(T):
        R[t, 0] = 0.02 + 0.3 * (next(g) - 0.5)
        R[t, 1] = 0.02 + 0.3 * (next(g) - 0.5)
        R[t, 2] = -0.2 + 0.8 * (1.0 if t % 2 else -1.0) + 0.02 * (next(g) - 0.5)
    mu = R.sum(axis=0) / T
    return R - mu[None, :], mu


def crra(gamma):
    return np.array([1.0, gamma / 2, gamma * (gamma + 1) / 6, gamma * (gamma + 1) * (gamma + 2) / 24])


def floor_sweep_ref(solve_fn, mu, c, nfloors=5, floors=None, mean_tol=1e-3, max_solves=16, warm_start=True):
    """Python mirror of the return-floor sweep (driver.cu floor_sweep; the
    paper's c1 calibration, PAPER.md:757 — not part of the reference code),
    driven by any solve_fn(coeffs, x0) -> x. Used to check the device sweep's
    decisions against CPU-oracle solves."""
    mu = np.asarray(mu, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    total = [0]

    def run(coeffs, x0):
        x = solve_fn(np.asarray(coeffs, dtype=np.float64), x0)
        total[0] += 1
        return {"c1": float(coeffs[0]), "mean": float(mu @ x), "x": x}

    mv = run([0.0, c[1], 0.0, 0.0], None)
    m_mv, m_max = mv["mean"], float(np.max(mu))
    span = m_max - m_mv
    fl = list(floors) if floors is not None else [m_mv + span * k / (nfloors + 1) for k in range(1, nfloors + 1)]
    tol = mean_tol * max(abs(span), 1e-300)
    cache = []

    def ev(c1, used):
        for e in cache:
            if e["c1"] == c1:
                return e
        x0 = None
        if warm_start and cache:
            nb = cache[0]
            for e in cache:
                if abs(e["c1"] - c1) < abs(nb["c1"] - c1):
                    nb = e
            x0 = nb["x"]
        cache.append(run([c1, c[1], c[2], c[3]], x0))
        used[0] += 1
        return cache[-1]

    c1_start = c[0] if c[0] > 0 else 1.0
    best, solves = [], []
    for r in fl:
        used = [0]
        ev(0.0, used)

        def closest():
            b = None
            for e in cache:
                if b is None or abs(e["mean"] - r) < abs(b["mean"] - r) or (
                        abs(e["mean"] - r) == abs(b["mean"] - r) and e["c1"] < b["c1"]):
                    b = e
            return b

        def bracket():
            lo, hi, have = 0.0, 0.0, False
            for e in cache:
                if e["mean"] < r and e["c1"] > lo:
                    lo = e["c1"]
                if e["mean"] >= r and (not have or e["c1"] < hi):
                    hi, have = e["c1"], True
            return lo, hi, have

        lo, hi, have = bracket()
        probe = max([c1_start] + [e["c1"] for e in cache])
        while not have and used[0] < max_solves and probe < 1e15:
            e = ev(probe, used)
            if e["mean"] >= r:
                break
            probe *= 2.0
            lo, hi, have = bracket()
        lo, hi, have = bracket()
        while have and used[0] < max_solves and abs(closest()["mean"] - r) > tol and hi - lo > 1e-12 * hi:
            ev(0.5 * (lo + hi), used)
            lo, hi, have = bracket()
        best.append(closest())
        solves.append(used[0])
    return {"floors": fl, "best": best, "solves": solves, "m_mv": m_mv, "m_max": m_max, "total": total[0]}
