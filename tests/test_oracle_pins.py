"""Pins the CPU parity oracle (oracle/, a C++ restatement of the reference)
against every known-answer constant and relational test the reference suite
holds for the hot path. Each test cites the reference test it re-expresses
(/root/reference/proj/tests/...). CPU only."""
import math

import numpy as np
import pytest

from oracle import pyoracle as po
from tests import refhelpers as rh


# ---- test_rng.cpp ------------------------------------------------------------
def test_splitmix64_published_stream():  # test_rng.cpp:7-17
    assert list(po.splitmix(0, "u64", 3)) == [16294208416658607535, 7960286522194355700, 487617019471545679]
    assert list(po.splitmix(1234567, "u64", 3)) == [6457827717110365317, 3203168211198807973,
                                                    9817491932198370423]


def test_splitmix_unit_top53():  # test_rng.cpp:19-25
    u = po.splitmix(42, "unit", 4)
    np.testing.assert_allclose(u, [0.74156487877182331, 0.1599103928769201, 0.27860113025513866,
                                   0.34419071652363753], rtol=1e-15)


def test_splitmix_uniform_normal_sign():  # test_rng.cpp:27-64
    u = po.splitmix(9, "uniform", 1000, -0.1, 0.4)
    assert np.all(u >= -0.1) and np.all(u < 0.4)
    assert np.array_equal(u, po.splitmix(9, "uniform", 1000, -0.1, 0.4))
    g = po.splitmix(7, "normal", 200000)
    assert abs(g.mean()) < 0.01 and abs((g * g).mean() - 1) < 0.02
    s = po.splitmix(11, "sign", 100000)
    assert set(np.unique(s)) <= {-1.0, 1.0}
    assert 49000 < (s > 0).sum() < 51000


# ---- test_panel.cpp ----------------------------------------------------------
def test_center_panel_and_validation():  # test_panel.cpp:5-36
    R = np.array([[0.1, 0.2], [0.3, -0.1], [0.2, 0.5]])
    A, mu = po.center_panel(R)
    assert abs(mu[0] - 0.2) <= 1e-16 and abs(mu[1] - 0.2) <= 1e-16
    assert np.all(np.abs(A.sum(axis=0)) < 1e-14)
    np.testing.assert_allclose(A + mu[None, :], R, atol=1e-15)
    with pytest.raises(po.OracleError) as e:
        po.center_panel(np.zeros((1, 3)))
    assert e.value.kind == "dimension_error"
    bad = np.zeros((3, 2))
    bad[1, 1] = np.nan
    with pytest.raises(po.OracleError) as e:
        po.center_panel(bad)
    assert e.value.kind == "data_error"


def test_crra_known_answers():  # test_panel.cpp:38-51, 53-60
    np.testing.assert_allclose(po.crra(1.0), [1.0, 0.5, 1 / 3, 0.25], rtol=1e-15)
    assert list(po.crra(2.0)) == [1.0, 1.0, 1.0, 1.0]
    for bad in (0.0, -2.0):
        with pytest.raises(po.OracleError):
            po.crra(bad)
    with pytest.raises(po.OracleError):
        po.make_coefficients(-1, 0, 0, 1)
    with pytest.raises(po.OracleError):
        po.make_coefficients(0, 0, 0, 0)
    po.make_coefficients(0, 1, 0, 0)


# ---- test_oracle.cpp ---------------------------------------------------------
PROFILES = [np.array([10, 1, 10, 1.0]), np.array([1, 10, 1, 10.0]), np.array([10, 10, 10, 10.0]),
            rh.crra(6.0)]


def test_value_matches_plain_loops():  # test_oracle.cpp:29-43
    for seed in range(5):
        A, mu = rh.lcg_panel(4 + seed % 3, 15, seed)
        x = rh.simplex_point(A.shape[1], seed + 100)
        for c in PROFILES:
            o = po.CpuOracle(A, mu, c)
            cache = o.make_cache(x)
            ref = rh.ref_value(A, mu, c, x)
            assert abs(o.value(cache) - ref) <= 1e-13 * (1 + abs(ref))


def test_moments_recombine():  # test_oracle.cpp:45-57
    A, mu = rh.lcg_panel(5, 30, 3)
    c = rh.crra(4.0)
    o = po.CpuOracle(A, mu, c)
    x = rh.simplex_point(5, 7)
    cache = o.make_cache(x)
    m1, m2, m3, m4 = o.moments(cache)
    assert m1 == pytest.approx(mu @ x, rel=1e-14)
    assert m2 >= 0 and m4 >= 0
    assert o.value(cache) == pytest.approx(-c[0] * m1 + c[1] * m2 - c[2] * m3 + c[3] * m4, rel=1e-13)


def test_gradient_loops_and_fd():  # test_oracle.cpp:59-77
    for seed in range(8):
        A, mu = rh.lcg_panel(3 + seed % 4, 12 + 3 * seed, seed)
        c = rh.crra(2.0 + seed) if seed % 2 else np.array([10, 10, 10, 10.0])
        o = po.CpuOracle(A, mu, c)
        x = rh.simplex_point(A.shape[1], seed + 9)
        g = o.gradient(o.make_cache(x))
        gl = rh.loop_gradient(A, mu, c, x)
        assert np.max(np.abs(g - gl)) <= 1e-13 * (1 + np.max(np.abs(gl)))
        h = 1e-6 * (1 + np.max(np.abs(x)))
        gf = rh.fd_gradient(lambda y: rh.ref_value(A, mu, c, y), x, h)
        assert np.max(np.abs(g - gf)) <= 1e-6 * (1 + np.max(np.abs(gf)))


def test_hvp_vs_fd():  # test_oracle.cpp:79-98
    for seed in range(6):
        A, mu = rh.lcg_panel(4, 20, 40 + seed)
        c = rh.crra(6.0)
        o = po.CpuOracle(A, mu, c)
        x = rh.simplex_point(4, seed)
        v = np.zeros(4)
        v[seed % 4] = 1.0
        v[(seed + 1) % 4] = -0.5
        hv = o.hvp(o.make_cache(x), v)
        h = 1e-6 * (1 + np.max(np.abs(x)))
        hv_fd = rh.fd_directional(lambda y: rh.loop_gradient(A, mu, c, y), x, v, h)
        assert np.max(np.abs(hv - hv_fd)) <= 1e-6 * (1 + np.max(np.abs(hv_fd)))


def test_third_action_vs_fd_and_symmetry():  # test_oracle.cpp:100-124
    A, mu = rh.lcg_panel(5, 25, 77)
    c = rh.crra(6.0)
    o = po.CpuOracle(A, mu, c)
    x = rh.simplex_point(5, 11)
    u = np.array([1, -1, 0.5, 0, -0.5])
    v = np.array([0.2, 0.3, -0.1, 0.4, -0.8])
    cache = o.make_cache(x)
    tuv = o.third_action(cache, u, v)
    fd = rh.fd_directional(lambda y: o.hvp(o.make_cache(y), u), x, v, 1e-5)
    assert np.max(np.abs(tuv - fd)) <= 1e-5 * (1 + np.max(np.abs(fd)))
    tvu = o.third_action(cache, v, u)
    assert np.max(np.abs(tuv - tvu)) <= 1e-14 * (1 + np.max(np.abs(tuv)))


def test_pass_count_contract():  # test_oracle.cpp:126-154
    A, mu = rh.lcg_panel(6, 18, 5)
    o = po.CpuOracle(A, mu, rh.crra(4.0))
    x = rh.simplex_point(6, 2)
    v = rh.simplex_point(6, 3)
    cache = o.make_cache(x)
    assert o.passes() == (1, 0)
    o.value(cache)
    assert sum(o.passes()) == 1
    o.gradient(cache)
    assert o.passes() == (1, 1)
    o.gradient(cache)
    assert sum(o.passes()) == 2
    o.reset_passes()
    o.hvp(cache, v)
    assert sum(o.passes()) == 2
    o.reset_passes()
    o.third_action(cache, v, x)
    assert sum(o.passes()) == 3


def test_face_oracle_reproduces_full():  # test_oracle.cpp:156-186
    tau = 1e-8
    A, mu = rh.lcg_panel(6, 20, 9)
    c = rh.crra(6.0)
    full = po.CpuOracle(A, mu, c)
    x = np.array([0.3, tau, 0.25, 0.2, tau, 0.25 - 2 * tau])
    assert abs(x.sum() - 1) < 1e-15
    idx, zoff, mu_pin, _ = po.restrict_to_face(A, mu, x, tau)
    assert list(idx) == [0, 2, 3, 5]
    face = po.CpuOracle(A[:, idx], mu[idx], c, zoff=zoff, value_offset=-c[0] * mu_pin)
    cf, cr = full.make_cache(x), face.make_cache(x[idx])
    assert abs(face.value(cr) - full.value(cf)) <= 1e-12 * (1 + abs(full.value(cf)))
    np.testing.assert_allclose(face.gradient(cr), full.gradient(cf)[idx], rtol=1e-12)


def test_diag_weights_and_sample_direction():  # test_oracle.cpp:188-206
    A, mu = rh.lcg_panel(4, 10, 21)
    c = rh.crra(6.0)
    o = po.CpuOracle(A, mu, c)
    x = rh.simplex_point(4, 4)
    w = o.hessian_diag_weights(o.make_cache(x))
    z = A @ x
    np.testing.assert_allclose(w, 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z, rtol=1e-14)
    d = np.array([1, -1, 0, 0.0])
    assert np.max(np.abs(o.sample_direction(d) - A @ d)) <= 1e-15


def test_typed_errors():  # test_oracle.cpp:208-225
    A, mu = rh.lcg_panel(4, 10, 1)
    c = rh.crra(2.0)
    with pytest.raises(po.OracleError) as e:
        po.oracle_create_mu(A, np.zeros(3))
    assert e.value.kind == "dimension_error"
    o = po.CpuOracle(A, mu, c)
    with pytest.raises(po.OracleError) as e:
        o.make_cache(np.zeros(5))
    assert e.value.kind == "dimension_error"
    wild = po.CpuOracle(np.full((4, 2), 1e200), np.zeros(2), c)
    with pytest.raises(po.OracleError) as e:
        wild.make_cache(np.array([1.0, 0.0]))
    assert e.value.kind == "numeric_error"


# ---- test_linesearch.cpp -----------------------------------------------------
def test_power_sums_worked_example():  # test_linesearch.cpp:9-23
    assert list(po.power_sums([2.0], [3.0])) == [6, 12, 24, 9, 18, 36, 27, 54, 81]


def test_power_sums_hand_loop():  # test_linesearch.cpp:25-44
    r = po.splitmix(17, "unit", 26)
    # SplitMix64(17) uniform draws interleaved z, w as in the reference loop
    z = -1 + 2 * r[0::2]
    w = -1 + 2 * r[1::2]
    s = po.power_sums(z, w)
    assert s[5] == pytest.approx(np.sum(z * z * w * w) / 13, rel=1e-14)
    assert s[7] == pytest.approx(np.sum(z * w ** 3) / 13, rel=1e-14)
    assert s[8] == pytest.approx(np.sum(w ** 4) / 13, rel=1e-14)
    with pytest.raises(po.OracleError):
        po.power_sums(z, np.zeros(14))


def test_quartic_model_reproduces_objective():  # test_linesearch.cpp:46-72
    for seed in range(6):
        A, mu = rh.lcg_panel(5, 20, seed)
        c = rh.crra(6.0) if seed % 2 else np.array([10, 10, 10, 10.0])
        o = po.CpuOracle(A, mu, c)
        x = rh.simplex_point(5, seed + 30, 1e-3)
        d = po.splitmix(seed + 200, "uniform", 5, -1.0, 1.0)
        d -= d.mean()
        cache = o.make_cache(x)
        cap = po.alpha_max(x, d, 0.0)
        m = o.line_model(cache, d, cap)
        assert m[0] == o.value(cache)
        assert m[1] == pytest.approx(o.gradient(cache) @ d, rel=1e-12)
        for k in range(21):
            al = cap * k / 20
            direct = rh.ref_value(A, mu, c, x + al * d)
            ev = m[0] + al * (m[1] + al * (m[2] + al * (m[3] + al * m[4])))
            assert abs(ev - direct) <= 1e-12 * (1 + abs(direct))


def test_line_model_rejects_bad_directions():  # test_linesearch.cpp:74-81
    A, mu = rh.lcg_panel(4, 10, 3)
    o = po.CpuOracle(A, mu, rh.crra(2.0))
    cache = o.make_cache(rh.simplex_point(4, 1))
    for d in (np.zeros(4), np.ones(4)):
        with pytest.raises(po.OracleError) as e:
            o.line_model(cache, d, 1.0)
        assert e.value.kind == "domain_error"


def test_exact_quartic_beats_grid():  # test_linesearch.cpp:83-109
    for seed in range(10):
        n = 4 + seed % 3
        A, mu = rh.lcg_panel(n, 16, seed + 60)
        o = po.CpuOracle(A, mu, rh.crra(4.0 + seed))
        x = rh.simplex_point(n, seed + 90, 1e-4)
        d = po.splitmix(seed + 400, "uniform", n, -1.0, 1.0)
        d -= d.mean()
        cache = o.make_cache(x)
        cap = po.alpha_max(x, d, 1e-4)
        if not math.isfinite(cap):
            cap = 1.0
        m = o.line_model(cache, d, cap)
        a_star, f_star = po.minimize_line(m[:5], cap)
        ev = lambda a: m[0] + a * (m[1] + a * (m[2] + a * (m[3] + a * m[4])))
        assert 0 <= a_star <= cap
        assert f_star == pytest.approx(ev(a_star), abs=1e-14)
        _, f_grid = rh.grid_line_min(ev, cap)
        assert f_star <= f_grid + 1e-12 * (1 + abs(f_grid))


def test_minimizer_degenerate_shapes():  # test_linesearch.cpp:111-148
    a, f = po.minimize_line([1.0, -2.0, 1.0, 0, 0], 5.0)
    assert a == pytest.approx(1.0, rel=1e-14) and abs(f) <= 1e-14
    a, f = po.minimize_line([0.0, -1.0, 0, 0, 0], 2.0)
    assert a == 2.0 and f == pytest.approx(-2.0, rel=1e-14)
    assert po.minimize_line([3.0, 4.0, 1.0, 0, 0], 1.0) == (0.0, 3.0)
    assert po.minimize_line([7.0, 0, 0, 0, 0], 0.0) == (0.0, 7.0)


def test_cubic_roots_all_branches():  # test_linesearch.cpp:150-169
    r3 = np.sort(po.cubic_real_roots(1, -6, 11, -6))
    np.testing.assert_allclose(r3, [1, 2, 3], rtol=1e-10)
    r1 = po.cubic_real_roots(1, 0, 1, 1)
    assert r1.size == 1 and abs(r1[0] ** 3 + r1[0] + 1) < 1e-12
    rt = po.cubic_real_roots(1, -6, 12, -8)
    assert rt.size > 0 and np.all(np.abs(rt - 2) <= 2e-6)


def test_armijo():  # test_linesearch.cpp:171-190
    phi = lambda a: -a + a * a
    a, st = po.armijo_search(phi, -1.0, 1.0, 0.5, 0.5)
    assert not st and a == pytest.approx(0.5, abs=1e-15)
    a, st = po.armijo_search(phi, -1.0, 0.9)
    assert a == pytest.approx(0.9, abs=1e-15)
    a, st = po.armijo_search(lambda a: a, -1.0, 1.0)
    assert st and a == 0.0
    with pytest.raises(po.OracleError):
        po.armijo_search(phi, 1.0, 1.0)
    with pytest.raises(po.OracleError):
        po.armijo_search(phi, -1.0, 1.0, 2.0, 0.5)


# ---- test_simplex.cpp --------------------------------------------------------
def _dense_U(n):
    return np.stack([po.basis_apply(n, np.eye(n - 1)[j]) for j in range(n - 1)], axis=1)


def test_tangent_basis_orthonormal():  # test_simplex.cpp:10-20, 22-36
    for n in (2, 3, 5, 17, 64):
        U = _dense_U(n)
        assert np.max(np.abs(U.T @ U - np.eye(n - 1))) < 1e-14
        assert np.max(np.abs(U.T @ np.ones(n))) < 1e-14
    n = 9
    U = _dense_U(n)
    y, x = rh.simplex_point(n - 1, 3), rh.simplex_point(n, 4)
    assert np.max(np.abs(po.basis_apply(n, y) - U @ y)) < 1e-14
    assert np.max(np.abs(po.basis_apply_transpose(n, x) - U.T @ x)) < 1e-14


def test_projection_worked_examples():  # test_simplex.cpp:66-88
    np.testing.assert_allclose(po.project_slice([2, -1], 0.0), [1, 0], atol=1e-15)
    np.testing.assert_allclose(po.project_slice([0.6, 0.6, -0.2], 0.0), [0.5, 0.5, 0], atol=1e-15)
    v = np.array([0.2, 0.5, 0.3])
    assert np.max(np.abs(po.project_slice(v, 0.0) - v)) < 1e-15


def test_projection_variational():  # test_simplex.cpp:90-104, 106-110
    for seed in range(20):
        n = 2 + seed % 7
        v = 3.0 * po.splitmix(seed * 31 + 7, "uniform", n, -1.0, 1.0)
        tau = 0.0 if seed % 3 == 0 else 1e-3
        mass = 2.0 if seed % 4 == 0 else 1.0
        pr = po.project_slice(v, tau, mass)
        assert rh.is_valid_projection(v, pr, tau, mass)
        assert np.max(np.abs(po.project_slice(pr, tau, mass) - pr)) < 1e-12
    for tau in (0.3, -0.1):
        with pytest.raises(po.OracleError):
            po.project_slice(np.ones(4), tau)


def test_alpha_max():  # test_simplex.cpp:112-136
    assert po.alpha_max([0.5, 0.3, 0.2], [1.0, -0.5, -0.5], 0.1) == pytest.approx(0.2, abs=1e-15)
    assert math.isinf(po.alpha_max([0.5, 0.3, 0.2], [1, 1, 1.0], 0.0))
    for seed in range(10):
        n = 3 + seed % 5
        xs = rh.simplex_point(n, seed, 1e-4)
        dd = po.splitmix(seed + 50, "uniform", n, -1.0, 1.0)
        dd -= dd.mean()
        am = po.alpha_max(xs, dd, 1e-4)
        if math.isfinite(am) and am > 0:
            at = xs + am * dd
            assert at.min() >= 1e-4 - 1e-12
            assert at.min() <= 1e-4 + 1e-9 * am + 1e-12


def test_residuals():  # test_simplex.cpp:138-157
    assert po.projected_kkt_residual(np.full(5, 3.7)) < 1e-14
    assert po.projected_kkt_residual([1, 2, 3.0]) == pytest.approx(math.sqrt(2), rel=1e-14)
    x = np.array([1 - 2e-8, 1e-8, 1e-8])
    gb = np.array([0.0, 5.0, 5.0])
    assert po.projected_kkt_residual(gb) > 1
    assert po.gradient_mapping_residual(x, gb, 1e-8) < 1e-12


def test_face_restriction_bookkeeping():  # test_simplex.cpp:159-178
    tau = 1e-8
    A, mu = rh.lcg_panel(5, 12, 13)
    x = np.array([0.4, tau, 0.3, tau, 0.3 - 2 * tau])
    idx, zoff, mu_pin, free_mass = po.restrict_to_face(A, mu, x, tau)
    assert list(idx) == [0, 2, 4]
    assert free_mass == pytest.approx(1 - 2 * tau, rel=1e-15)
    assert np.max(np.abs(zoff - tau * (A[:, 1] + A[:, 3]))) < 1e-20
    assert mu_pin == pytest.approx(tau * (mu[1] + mu[3]), rel=1e-14)
    with pytest.raises(po.OracleError) as e:
        po.restrict_to_face(A, mu, np.full(5, tau), tau)
    assert e.value.kind == "domain_error"


# ---- test_affine_normal.cpp --------------------------------------------------
def test_householder_frame():  # test_affine_normal.cpp:9-42
    for seed in range(6):
        m = 2 + seed
        g = po.splitmix(seed + 5, "uniform", 2 * m, -1.0, 1.0)
        g, w = g[:m].copy(), g[m:]
        if seed == 2:
            g[0] = -g[0]
        nu, v, beta, gn = po.householder_frame(g)
        assert gn == pytest.approx(np.linalg.norm(g), rel=1e-14)
        assert np.linalg.norm(nu) == pytest.approx(1.0, rel=1e-14)
        Q = np.stack([po.frame_apply_Q(g, np.eye(m - 1)[k]) for k in range(m - 1)], axis=1)
        assert np.max(np.abs(Q.T @ Q - np.eye(m - 1))) < 1e-13
        assert np.max(np.abs(Q.T @ nu)) < 1e-13
        assert np.max(np.abs(po.frame_apply_Qt(g, w) - Q.T @ w)) < 1e-13
    with pytest.raises(po.OracleError):
        po.householder_frame(np.zeros(3))
    with pytest.raises(po.OracleError) as e:
        po.householder_frame([2.0])
    assert e.value.kind == "dimension_error"


def test_descent_identity_both_modes():  # test_affine_normal.cpp:44-73
    checked = 0
    for seed in range(25):
        n = 3 + seed % 6
        A, mu = rh.lcg_panel(n, 18 + seed, seed)
        c = np.array([10, 10, 10, 10.0]) if seed % 3 == 0 else rh.crra(2.0 + seed % 5)
        o = po.CpuOracle(A, mu, c)
        x = rh.simplex_point(n, seed + 71, 1e-6)
        cache = o.make_cache(x)
        g = o.gradient(cache)
        gn = np.linalg.norm(po.basis_apply_transpose(n, g))
        if not gn > 1e-12:
            continue
        dd, _ = o.yand_direction(cache, po.tangent_config("direct"), seed)
        assert abs(g @ dd + gn) <= 1e-10 * (1 + gn)
        assert abs(dd.sum()) <= 1e-12 * (1 + np.linalg.norm(dd))
        dp, _ = o.yand_direction(cache, po.tangent_config("pcg", lam=1e-4, krylov_maxit=2), seed)
        assert abs(g @ dp + gn) <= 1e-10 * (1 + gn)
        checked += 1
    assert checked >= 20


def test_direct_vs_exact_pcg():  # test_affine_normal.cpp:75-100
    n = 6
    A, mu = rh.lcg_panel(n, 30, 99)
    o = po.CpuOracle(A, mu, rh.crra(6.0))
    cache = o.make_cache(rh.simplex_point(n, 8, 1e-6))
    dd, ddiag = o.yand_direction(cache, po.tangent_config("direct"), 0)
    dp, pdiag = o.yand_direction(cache, po.tangent_config("pcg", lam=0.0, krylov_tol=1e-14, krylov_maxit=500,
                                                          exact_trace=True), 0)
    assert not ddiag.lambda_fallback
    assert pdiag.krylov_iters > 0
    assert np.max(np.abs(dd - dp)) <= 1e-9 * (1 + np.max(np.abs(dd)))


def test_two_asset_direction():  # test_affine_normal.cpp:102-119
    A, mu = rh.lcg_panel(2, 15, 4)
    o = po.CpuOracle(A, mu, rh.crra(4.0))
    cache = o.make_cache(np.array([0.6, 0.4]))
    g = o.gradient(cache)
    gbar = po.basis_apply_transpose(2, g)
    d, _ = o.yand_direction(cache, po.tangent_config("direct"))
    assert np.linalg.norm(d) == pytest.approx(1.0, rel=1e-12)
    assert g @ d == pytest.approx(-np.linalg.norm(gbar), rel=1e-12)


def test_cg_capped():  # test_affine_normal.cpp:121-144
    M = np.array([[4, 1, 0], [1, 3, 1], [0, 1, 2.0]])
    b = np.array([1, 2, 3.0])
    x, it, bd = po.cg_dense(M, b, 1e-14, 50)
    assert not bd and it <= 3 and np.max(np.abs(M @ x - b)) < 1e-10
    x, it, bd = po.cg_dense(-np.eye(3), b, 1e-14, 50)
    assert bd and np.all(np.isfinite(x))


def test_stationary_raises_domain_error():  # test_affine_normal.cpp:146-159
    o = po.CpuOracle(np.zeros((4, 2)), np.array([0.1, 0.2]), np.array([0, 1, 0, 0.0]))
    cache = o.make_cache(np.array([0.5, 0.5]))
    with pytest.raises(po.OracleError) as e:
        o.yand_direction(cache, po.tangent_config("direct"))
    assert e.value.kind == "domain_error"


# ---- test_solver.cpp ---------------------------------------------------------
def test_two_asset_mv_closed_form():  # test_solver.cpp:32-45
    for seed in (1, 2, 3, 9):
        A, mu = rh.lcg_panel(2, 40, seed)
        cfg = po.preset("small")
        cfg.epsilon = 1e-10
        xs, rep = po.solve(A, mu, [1, 1, 0, 0], cfg)
        w, f = rh.mv_two_asset_optimum(A, mu, 1.0, 1.0, cfg.tau)
        assert rep.status == 0
        assert abs(xs[0] - w) <= 1e-7
        assert abs(rep.f_star - f) <= 1e-12


def test_small_preset_converges():  # test_solver.cpp:47-70 (minus the PG baseline)
    for seed in range(4):
        n = 5 + 3 * seed
        A, mu = rh.lcg_panel(n, 60, seed + 7)
        c = rh.crra(4.0 + seed)
        cfg = po.preset("small")
        xs, rep = po.solve(A, mu, c, cfg)
        assert rep.status == 0
        assert rep.kkt_residual <= cfg.epsilon
        assert xs.min() >= cfg.tau - 1e-15
        assert abs(xs.sum() - 1) < 1e-12
        assert rep.f_star == pytest.approx(rh.ref_value(A, mu, c, xs), rel=1e-13)
        assert rep.oracle_passes > 0 and rep.config_label == b"small"


def test_solves_deterministic():  # test_solver.cpp:72-84
    A, mu = rh.lcg_panel(12, 80, 3)
    c = rh.crra(6.0)
    for label in ("small", "large"):
        x1, r1 = po.solve(A, mu, c, po.preset(label))
        x2, r2 = po.solve(A, mu, c, po.preset(label))
        assert r1.f_star == r2.f_star and np.array_equal(x1, x2)
        assert r1.iterations == r2.iterations and r1.oracle_passes == r2.oracle_passes


def test_observer_trajectory_and_dominated_pin():  # test_solver.cpp:86-119
    A, mu = rh.dominated_panel(50)
    c = rh.crra(6.0)
    cfg = po.preset("small")
    trace = []
    xs, rep = po.solve(A, mu, c, cfg, observer=lambda it, f, x: trace.append((it, f, x)))
    assert trace and trace[0][0] == 0
    for k, (it, f, x) in enumerate(trace):
        assert x.min() >= cfg.tau - 1e-12 and abs(x.sum() - 1) <= 1e-12
        if k:
            assert f <= trace[k - 1][1] + 1e-12 * (1 + abs(trace[k - 1][1]))
            assert it > trace[k - 1][0]
    assert trace[-1][1] >= rep.f_star - 1e-12 * (1 + abs(rep.f_star))
    A, mu = rh.dominated_panel(60)
    xs, rep = po.solve(A, mu, c, cfg)
    assert rep.status == 0 and rep.face_events >= 1
    assert xs[2] == cfg.tau and xs[0] > 0.1 and xs[1] > 0.1


def test_single_asset_and_budget():  # test_solver.cpp:121-152
    R = np.array([[0.1], [-0.05], [0.2], [0.0], [0.05]])
    A, mu = rh.center(R)
    xs, rep = po.solve(A, mu, rh.crra(2.0), po.preset("small"))
    assert rep.status == 0 and list(xs) == [1.0] and rep.kkt_residual == 0.0
    A, mu = rh.lcg_panel(10, 60, 5)
    c = rh.crra(8.0)
    tiny = po.preset("small")
    tiny.max_iter = 1
    tiny.epsilon = 1e-14
    xs, r1 = po.solve(A, mu, c, tiny)
    assert r1.status in (1, 2) and r1.iterations <= 1
    timed = po.preset("small")
    timed.has_max_elapsed = 1
    timed.max_elapsed_seconds = 0.0
    timed.epsilon = 1e-14
    xs, r2 = po.solve(A, mu, c, timed)
    assert r2.status == 3
    assert abs(xs.sum() - 1) < 1e-12
    assert r2.f_star == pytest.approx(rh.ref_value(A, mu, c, xs), rel=1e-13)


def test_solver_validation():  # test_solver.cpp:154-176
    A, mu = rh.lcg_panel(4, 20, 8)
    c = rh.crra(2.0)
    bad = po.preset("small")
    bad.epsilon = 0.0
    with pytest.raises(po.OracleError):
        po.solve(A, mu, c, bad)
    bad = po.preset("small")
    bad.tau = 0.3
    with pytest.raises(po.OracleError):
        po.solve(A, mu, c, bad)
    for x0 in (np.full(3, 1 / 3), np.full(4, 0.3), np.array([0.5, 0.7, -0.1, -0.1])):
        with pytest.raises(po.OracleError):
            po.solve(A, mu, c, po.preset("small"), x0=x0)
    with pytest.raises(po.OracleError):
        po.preset("medium")


def test_custom_start_and_spg_preamble():  # test_solver.cpp:178-197
    A, mu = rh.lcg_panel(6, 40, 11)
    c = rh.crra(6.0)
    cfg = po.preset("small")
    _, r1 = po.solve(A, mu, c, cfg, x0=rh.simplex_point(6, 77, cfg.tau))
    _, r2 = po.solve(A, mu, c, cfg)
    assert r1.status == 0
    assert abs(r1.f_star - r2.f_star) <= 1e-9 * (1 + abs(r1.f_star))
    A, mu = rh.dominated_panel(80)
    cfg = po.preset("large")
    xs, rep = po.solve(A, mu, c, cfg)
    assert rep.identification_steps > 0 and rep.status == 0 and xs[2] == cfg.tau
