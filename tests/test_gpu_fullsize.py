"""Parity at BASELINE.json's full sizes: C4 (n=5000, T=5000) and C5 (n=4096,
T=262144, 8 GiB) against the CPU oracle on the very same bits (the C5 panel is
generated on the device and copied back), at the 1e-11 bar, plus
size-independent identities of the exact oracle on C5 (linearity and symmetry
of the Hessian, symmetry of the third action, a1 = g'd of the line model)."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def _close(a, b, scale, rel=1e-11):
    err = float(np.max(np.abs(np.asarray(a) - np.asarray(b))))
    ref = max(float(np.max(np.abs(b))), scale)
    assert err <= rel * ref, (err, ref)


def _scales(A, c, x, V):
    T = A.shape[0]
    z = A @ x
    absA = np.abs(A)
    w = np.abs(2 * c[1] * z - 3 * c[2] * z * z + 4 * c[3] * z ** 3) / T
    psi2 = np.abs(2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z)
    g_s = float(np.max(absA.T @ w))
    h_s = [float(np.max(absA.T @ (psi2 * np.abs(A @ v)) / T)) for v in V]
    return g_s, h_s


def test_c4_full_size_parity():
    from paper_2604_25378_b200.datagen import make_panel, random_simplex_point, random_tangents
    from paper_2604_25378_b200.gpu_oracle import GpuOracle
    A, mu, c = make_panel("C4", seed=2)
    n = A.shape[1]
    x = random_simplex_point(n, 5)
    V = random_tangents(n, 8, 5)
    po.set_threads(os.cpu_count() or 1)
    try:
        cpu = po.CpuOracle(A, mu, c)
        cc = cpu.make_cache(x)
        gpu = GpuOracle(A, mu, c)
        gc = gpu.make_cache(x)
        g_s, h_s = _scales(A, c, x, V[:2])
        _close(gpu.value(gc), cpu.value(cc), 0.0)
        _close(gpu.gradient(gc), cpu.gradient(cc), g_s)
        H = gpu.hvp(gc, V)  # 8 RHS: tensor-core cluster path
        for i in range(2):
            _close(H[i], cpu.hvp(cc, V[i]), h_s[i])
        lm = gpu.line_model(gc, V[0], 1.0)
        np.testing.assert_allclose([lm.a0, lm.a1, lm.a2, lm.a3, lm.a4], cpu.line_model(cc, V[0], 1.0)[:5],
                                   rtol=1e-11, atol=1e-15)
    finally:
        po.set_threads(1)


def test_c5_full_size_parity_and_identities():
    torch = pytest.importorskip("torch")
    from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, random_tangents, raw_returns
    from paper_2604_25378_b200.gpu_oracle import GpuOracle
    spec = CONFIGS["C5"]
    T, n = spec.T, spec.n
    X = raw_returns(spec, 77, device="cuda")
    mu_t = X.sum(0) / T
    X.sub_(mu_t)
    c = crra(spec.gamma)
    mu = mu_t.cpu().numpy()
    gpu = GpuOracle(None, mu, c, device_panel=(X.data_ptr(), n, T, n))
    x = random_simplex_point(n, 9)
    V = random_tangents(n, 8, 9)
    gc = gpu.make_cache(x)
    g = gpu.gradient(gc)
    H = gpu.hvp(gc, V)
    H1 = gpu.hvp(gc, V[0])
    # size-independent identities of the exact oracle (no CPU needed)
    a, b = 0.7, -1.3
    Hab = gpu.hvp(gc, a * V[1] + b * V[2])
    assert np.max(np.abs(Hab - (a * H[1] + b * H[2]))) <= 1e-10 * np.max(np.abs(Hab))
    assert abs(V[3] @ H[4] - V[4] @ H[3]) <= 1e-10 * abs(V[3] @ H[4])
    T34 = gpu.third_action(gc, V[3], V[4])
    T43 = gpu.third_action(gc, V[4], V[3])
    assert np.max(np.abs(T34 - T43)) <= 1e-12 * np.max(np.abs(T34))
    lm = gpu.line_model(gc, V[0], 1.0)
    assert lm.a1 == pytest.approx(g @ V[0], rel=1e-11)
    assert np.max(np.abs(H[0] - H1)) <= 1e-11 * np.max(np.abs(H1))  # tensor-core vs streaming path
    # 4-RHS and 8-pair third-action tensor-core paths vs the single streaming pass
    H4 = gpu.hvp(gc, V[4:])
    assert np.max(np.abs(H4 - H[4:])) <= 1e-11 * np.max(np.abs(H[4:]))
    W = V[::-1].copy()
    T8 = gpu.third_action(gc, V, W)
    for i in (0, 5):
        Ti = gpu.third_action(gc, V[i], W[i])
        assert np.max(np.abs(T8[i] - Ti)) <= 1e-11 * np.max(np.abs(Ti))
    T4 = gpu.third_action(gc, V[:4], W[:4])
    assert np.max(np.abs(T4 - T8[:4])) <= 1e-11 * np.max(np.abs(T8[:4]))
    lm8 = np.array([lm.a0, lm.a1, lm.a2, lm.a3, lm.a4, *lm.sums])
    G = gpu.weighted_gram(gc)  # DMMA Gram over the full 8 GiB panel
    # the same bits on the CPU oracle (all host threads, test-only): every
    # tensor-core multi-RHS result, the line model and the Gram, not just one HVP
    A = X.cpu().numpy()
    del X
    po.set_threads(os.cpu_count() or 1)
    try:
        cpu = po.CpuOracle(A, mu, c)
        cc = cpu.make_cache(x)
        g_s, h_s = _scales(A, c, x, V)
        _close(gpu.value(gc), cpu.value(cc), 0.0)
        _close(g, cpu.gradient(cc), g_s)
        _close(H1, cpu.hvp(cc, V[0]), h_s[0])
        Hc = [cpu.hvp(cc, V[i]) for i in range(8)]
        for i in range(8):  # 8-RHS tensor-core HVP
            _close(H[i], Hc[i], h_s[i])
        z = A @ x
        psi3 = np.abs(-6 * c[2] + 24 * c[3] * z)
        absA = np.abs(A)
        for i in range(8):  # 8-pair tensor-core third action
            t_s = float(np.max(absA.T @ (psi3 * np.abs(A @ V[i]) * np.abs(A @ W[i])) / T))
            _close(T8[i], cpu.third_action(cc, V[i], W[i]), t_s)
        del absA
        lmc = cpu.line_model(cc, V[0], 1.0)  # a0..a4 and the nine power sums
        np.testing.assert_allclose(lm8, lmc, rtol=1e-11, atol=1e-15 * np.max(np.abs(lmc)))
        # Gram: G v = H v for every tangent v (the same contraction, oracle.hpp:92-101
        # vs affine_normal.hpp:169), and exact entries G_ij = sum psi''_t a_ti a_tj / T
        for i in range(8):
            _close(G @ V[i], Hc[i], h_s[i])
        psi2 = cpu.hessian_diag_weights(cc)
        rng = np.random.default_rng(3)
        for i, j in rng.integers(0, n, size=(24, 2)):
            ref = float(np.dot(psi2 * A[:, i], A[:, j])) / T
            scale = float(np.dot(np.abs(psi2 * A[:, i]), np.abs(A[:, j]))) / T
            assert abs(G[i, j] - ref) <= 1e-11 * scale, (i, j, G[i, j], ref)
        np.testing.assert_array_equal(G, G.T)
    finally:
        po.set_threads(1)
