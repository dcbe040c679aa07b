"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs. Mirrors the reference's oracle tests (test_oracle.cpp,
test_linesearch.cpp) with the CPU restatement as the independent reference.

Tolerance (north_star): objective, gradient and HVP to 1e-11 relative. We use
  |gpu - cpu|_inf <= 1e-11 * max(|cpu|_inf, scale)
where `scale` is the magnitude of the summed terms (|A|^T |w| for the A^T w
products); the two sides sum the same terms in different orders, so that is
the floating-point error scale of the reference's own arithmetic."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests import refhelpers as rh

pytestmark = pytest.mark.gpu

REL = 1e-11


def _close(gpu, cpu, scale=0.0, rel=REL):
    gpu, cpu = np.asarray(gpu), np.asarray(cpu)
    ref = max(float(np.max(np.abs(cpu))) if cpu.size else 0.0, float(scale))
    err = float(np.max(np.abs(gpu - cpu))) if cpu.size else 0.0
    assert err <= rel * ref + 1e-300, f"err {err:.3e} > {rel:g} * {ref:.3e}"


def _gpu(A, mu, c, **kw):
    from paper_2604_25378_b200.gpu_oracle import GpuOracle
    return GpuOracle(A, mu, c, **kw)


def _absscale(A, w):
    return float(np.max(np.abs(A).T @ np.abs(w)))


PANELS = [(4, 15, 0), (5, 30, 3), (7, 33, 5), (9, 64, 11), (2, 40, 1), (1, 6, 2), (33, 257, 4), (130, 700, 6)]


@pytest.mark.parametrize("n,T,seed", PANELS)
@pytest.mark.parametrize("prof", [0, 1, 2, 3])
def test_value_gradient_moments(n, T, seed, prof):
    c = [np.array([10, 1, 10, 1.0]), np.array([1, 10, 1, 10.0]), np.array([10, 10, 10, 10.0]), rh.crra(6.0)][prof]
    A, mu = rh.lcg_panel(n, T, seed)
    x = rh.simplex_point(n, seed + 100)
    cpu = po.CpuOracle(A, mu, c)
    gpu = _gpu(A, mu, c)
    cc, gc = cpu.make_cache(x), gpu.make_cache(x)
    _close(gpu.value(gc), cpu.value(cc))
    np.testing.assert_allclose(gpu.moments(gc), cpu.moments(cc), rtol=1e-11, atol=1e-300)
    z = A @ x
    w = (2 * c[1] * z - 3 * c[2] * z * z + 4 * c[3] * z ** 3) / T
    _close(gpu.gradient(gc), cpu.gradient(cc), _absscale(A, w))
    assert abs(gpu.value(gc) - rh.ref_value(A, mu, c, x)) <= 1e-13 * (1 + abs(rh.ref_value(A, mu, c, x)))


@pytest.mark.parametrize("n,T,seed", PANELS)
def test_hvp_third_weights_direction(n, T, seed):
    c = rh.crra(6.0)
    A, mu = rh.lcg_panel(n, T, seed)
    x = rh.simplex_point(n, seed)
    cpu, gpu = po.CpuOracle(A, mu, c), _gpu(A, mu, c)
    cc, gc = cpu.make_cache(x), gpu.make_cache(x)
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((8, n))
    z = A @ x
    psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
    for k in (1, 2, 3, 4, 8):
        H = gpu.hvp(gc, V[:k])
        for i in range(k):
            ref = cpu.hvp(cc, V[i])
            _close(H[i], ref, _absscale(A, psi2 * (A @ V[i]) / T))
    U = rng.standard_normal((3, n))
    T3 = gpu.third_action(gc, U, V[:3])
    psi3 = -6 * c[2] + 24 * c[3] * z
    for i in range(3):
        _close(T3[i], cpu.third_action(cc, U[i], V[i]), _absscale(A, psi3 * (A @ U[i]) * (A @ V[i]) / T))
    np.testing.assert_allclose(gpu.hessian_diag_weights(gc), cpu.hessian_diag_weights(cc), rtol=1e-13, atol=1e-15)
    d = V[0]
    _close(gpu.sample_direction(d), cpu.sample_direction(d), float(np.max(np.abs(A) @ np.abs(d))))


@pytest.mark.parametrize("n,T", [(4, 50), (64, 300), (100, 1000), (128, 513), (800, 2500), (4096, 700), (4500, 260),
                                 (5000, 333)])
def test_multi_rhs_cluster_paths(n, T):
    """k = 8 / 4 RHS go through the cluster column-split kernel (DSMEM exchange
    of partial row dots) whenever ld splits evenly; parity vs the CPU oracle."""
    c = rh.crra(10.0)
    rng = np.random.default_rng(n + T)
    A = rng.uniform(-0.1, 0.4, (T, n))
    mu = A.mean(axis=0)
    A = A - mu
    x = rng.exponential(size=n)
    x /= x.sum()
    cpu, gpu = po.CpuOracle(A, mu, c), _gpu(A, mu, c)
    cc, gc = cpu.make_cache(x), gpu.make_cache(x)
    z = A @ x
    psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
    psi3 = -6 * c[2] + 24 * c[3] * z
    U = rng.standard_normal((13, n))
    V = rng.standard_normal((13, n))
    for k in (8, 4, 13):
        H = gpu.hvp(gc, V[:k])
        T3 = gpu.third_action(gc, U[:k], V[:k])
        for i in range(k):
            _close(H[i], cpu.hvp(cc, V[i]), _absscale(A, psi2 * (A @ V[i]) / T))
            _close(T3[i], cpu.third_action(cc, U[i], V[i]), _absscale(A, psi3 * (A @ U[i]) * (A @ V[i]) / T))
    f0, t0, p0 = gpu.passes()
    gpu.hvp(gc, V[:8])
    f1, t1, p1 = gpu.passes()
    assert (f1 - f0, t1 - t0) == (8, 8)  # the reference contract: 2 logical passes per HVP


@pytest.mark.parametrize("n,T,seed", PANELS[:6])
def test_line_model(n, T, seed):
    if n < 2:
        pytest.skip("needs a tangent direction")
    c = rh.crra(6.0) if seed % 2 else np.array([10, 10, 10, 10.0])
    A, mu = rh.lcg_panel(n, T, seed)
    x = rh.simplex_point(n, seed + 30, 1e-3)
    d = po.splitmix(seed + 200, "uniform", n, -1.0, 1.0)
    d -= d.mean()
    cpu, gpu = po.CpuOracle(A, mu, c), _gpu(A, mu, c)
    cc, gc = cpu.make_cache(x), gpu.make_cache(x)
    cap = po.alpha_max(x, d, 0.0)
    mc = cpu.line_model(cc, d, cap)
    mg = gpu.line_model(gc, d, cap)
    got = np.array([mg.a0, mg.a1, mg.a2, mg.a3, mg.a4, *mg.sums])
    np.testing.assert_allclose(got, mc, rtol=1e-11, atol=1e-14 * np.max(np.abs(mc)))
    assert mg.a1 == pytest.approx(gpu.gradient(gc) @ d, rel=1e-11)
    from paper_2604_25378_b200.gpu_oracle import DomainError
    with pytest.raises(DomainError):
        gpu.line_model(gc, np.ones(n), 1.0)
    with pytest.raises(DomainError):
        gpu.line_model(gc, np.zeros(n), 1.0)


def test_line_models_batch_is_bitwise_the_single_calls():  # linesearch.hpp:62-81, solver.hpp:448-562
    """mvsk_gpu_line_models (the boundary ladder's rungs in one round trip) against k single line_model
    calls: identical bits, on a narrow panel (small-pass kernels), a C2-sized one and a face view; a
    non-tangent direction comes back marked instead of raising; k passes are counted."""
    for n, T, face in ((12, 60, False), (100, 400, False), (100, 400, True)):
        A, mu = rh.lcg_panel(n, T, 3)
        gpu = _gpu(A, mu, rh.crra(5.0))
        if face:
            free = np.arange(0, n, 2)
            gpu.set_face(free, 1e-4)
            x = np.full(free.size, (1.0 - 1e-4 * (n - free.size)) / free.size)
            m = free.size
        else:
            x = rh.simplex_point(n, 5, 1e-6)
            m = n
        gc = gpu.make_cache(x)
        rng = np.random.default_rng(7)
        D = rng.standard_normal((5, m))
        D -= D.mean(axis=1, keepdims=True)
        for rep in range(4):  # eager, capture and replay of the k-direction graph
            singles = [gpu.line_model(gc, D[i], 0.5) for i in range(5)]
            f0, t0, _ = gpu.passes()
            batch = gpu.line_models(gc, D, [0.5] * 5)
            assert gpu.passes()[0] - f0 == 5
            for a, b in zip(singles, batch):
                assert (a.a0, a.a1, a.a2, a.a3, a.a4) == (b.a0, b.a1, b.a2, b.a3, b.a4)
                assert np.array_equal(a.sums, b.sums)
        bad = D.copy()
        bad[2] += 1.0  # not tangent
        out = gpu.line_models(gc, bad, [0.5] * 5)
        assert np.isnan(out[2].a0) and all(np.isfinite(out[i].a0) for i in (0, 1, 3, 4))
        gpu.close()


def test_pass_count_contract():  # test_oracle.cpp:126-154
    A, mu = rh.lcg_panel(6, 18, 5)
    gpu = _gpu(A, mu, rh.crra(4.0))
    x, v = rh.simplex_point(6, 2), rh.simplex_point(6, 3)
    cache = gpu.make_cache(x)
    assert gpu.passes()[:2] == (1, 0)
    gpu.gradient(cache)
    assert gpu.passes()[:2] == (1, 1)
    gpu.gradient(cache)
    assert sum(gpu.passes()[:2]) == 2
    gpu.reset_passes()
    gpu.hvp(cache, v)
    assert sum(gpu.passes()[:2]) == 2 and gpu.passes()[2] == 1  # one physical pass
    gpu.reset_passes()
    gpu.third_action(cache, v, x)
    assert sum(gpu.passes()[:2]) == 3 and gpu.passes()[2] == 1


def test_face_view_matches_restricted_oracle():  # test_oracle.cpp:156-186
    tau = 1e-8
    A, mu = rh.lcg_panel(6, 20, 9)
    c = rh.crra(6.0)
    x = np.array([0.3, tau, 0.25, 0.2, tau, 0.25 - 2 * tau])
    idx, zoff, mu_pin, _ = po.restrict_to_face(A, mu, x, tau)
    face_cpu = po.CpuOracle(A[:, idx], mu[idx], c, zoff=zoff, value_offset=-c[0] * mu_pin)
    cr = face_cpu.make_cache(x[idx])
    gpu = _gpu(A, mu, c)
    gpu.set_face(idx, tau)
    gc = gpu.make_cache(x[idx])
    assert abs(gpu.value(gc) - face_cpu.value(cr)) <= 1e-12 * (1 + abs(face_cpu.value(cr)))
    np.testing.assert_allclose(gpu.gradient(gc), face_cpu.gradient(cr), rtol=1e-12)
    v = np.array([0.5, -0.2, 0.1, -0.4])
    np.testing.assert_allclose(gpu.hvp(gc, v), face_cpu.hvp(cr, v), rtol=1e-11)
    # the explicit zoff/value_offset constructor form (oracle.hpp:31-33)
    g2 = _gpu(A[:, idx], mu[idx], c)
    g2.set_offset(zoff, -c[0] * mu_pin)
    c2 = g2.make_cache(x[idx])
    assert abs(g2.value(c2) - face_cpu.value(cr)) <= 1e-13 * (1 + abs(face_cpu.value(cr)))
    np.testing.assert_allclose(g2.gradient(c2), face_cpu.gradient(cr), rtol=1e-12)


def test_typed_errors():  # test_oracle.cpp:208-225
    from paper_2604_25378_b200.gpu_oracle import DimensionError, NumericError
    A, mu = rh.lcg_panel(4, 10, 1)
    c = rh.crra(2.0)
    with pytest.raises(DimensionError):
        _gpu(A, np.zeros(3), c)
    g = _gpu(A, mu, c)
    with pytest.raises(DimensionError):
        g.make_cache(np.zeros(5))
    wild = _gpu(np.full((4, 2), 1e200), np.zeros(2), c)
    with pytest.raises(NumericError):
        wild.make_cache(np.array([1.0, 0.0]))


def test_weighted_gram_dmma():
    # 128 / 256: the full-tile kernel (psi'' precomputed by run_psi2), the others
    # the edge-tile kernel (psi'' in its load)
    for (n, T, seed) in [(20, 500, 1), (100, 1000, 2), (131, 777, 3), (300, 2000, 4), (128, 900, 5),
                         (256, 1500, 6)]:
        A, mu = rh.lcg_panel(n, T, seed) if n <= 33 else (np.random.default_rng(seed).uniform(-0.1, 0.4, (T, n)), None)
        if mu is None:
            A = A - A.mean(axis=0)
            mu = np.zeros(n)
        c = rh.crra(10.0)
        gpu = _gpu(A, mu, c)
        x = rh.simplex_point(n, seed)
        gc = gpu.make_cache(x)
        z = A @ x
        psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
        ref = (A * psi2[:, None]).T @ A / T
        G = gpu.weighted_gram(gc)
        scale = float(np.max((np.abs(A) * np.abs(psi2)[:, None]).T @ np.abs(A) / T))
        _close(G, ref, scale)
        assert np.array_equal(G, G.T)


def test_weighted_gram_variants_subprocess():
    """MVSK_GRAM_VAR (read once per process) selects the warp layout of the
    full-tile Gram kernel; variants 0 and 2 against fp64 numpy at n = 128."""
    import json
    import os
    import subprocess
    import sys
    code = (
        "import sys, json, numpy as np\n"
        "sys.path.insert(0, %r)\n"
        "from paper_2604_25378_b200.gpu_oracle import GpuOracle\n"
        "rng = np.random.default_rng(7); A = rng.uniform(-0.1, 0.4, (1000, 128)); A -= A.mean(0)\n"
        "c = np.array([1.0, 5.0, 55.0 / 3.0, 55.0]); x = np.full(128, 1 / 128)\n"
        "g = GpuOracle(A, np.zeros(128), c); G = g.weighted_gram(g.make_cache(x))\n"
        "z = A @ x; p2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z\n"
        "ref = (A * p2[:, None]).T @ A / 1000\n"
        "sc = float(np.max((np.abs(A) * np.abs(p2)[:, None]).T @ np.abs(A) / 1000))\n"
        "print(json.dumps({'err': float(np.max(np.abs(G - ref))) / sc, 'sym': bool(np.array_equal(G, G.T))}))\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for var in ("0", "2"):
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MVSK_GRAM_VAR=var),
                             capture_output=True, text=True, timeout=300, check=True)
        r = json.loads(out.stdout.strip().splitlines()[-1])
        assert r["err"] <= 1e-11 and r["sym"], (var, r)


def test_borrowed_panel_nonfinite_padding_is_rejected():
    """create_from_device reads whole ld-wide rows; NaN padding would turn into
    0 * NaN in every result, so it is rejected with a data error."""
    torch = pytest.importorskip("torch")
    from paper_2604_25378_b200.gpu_oracle import DataError, GpuOracle
    T, n, ld = 64, 9, 12
    rng = np.random.default_rng(1)
    A = rng.uniform(-0.1, 0.4, (T, n))
    A -= A.mean(0)
    buf = torch.full((T, ld), float("nan"), dtype=torch.float64, device="cuda")
    buf[:, :n] = torch.from_numpy(A).cuda()
    c = rh.crra(5.0)
    with pytest.raises(DataError):
        GpuOracle(None, np.zeros(n), c, device_panel=(buf.data_ptr(), ld, T, n))
    buf[:, n:] = 0.0
    g = GpuOracle(None, np.zeros(n), c, device_panel=(buf.data_ptr(), ld, T, n))
    x = rh.simplex_point(n, 2)
    cpu = po.CpuOracle(A, np.zeros(n), c)
    assert abs(g.value(g.make_cache(x)) - cpu.value(cpu.make_cache(x))) <= 1e-12
    g.close()


def test_datagen_configs_parity():
    from paper_2604_25378_b200.datagen import make_panel, random_simplex_point, random_tangents
    for name in ("C1", "C2", "C3"):
        A, mu, c = make_panel(name, seed=1)
        T, n = A.shape
        x = random_simplex_point(n, 3)
        V = random_tangents(n, 4, 3)
        cpu, gpu = po.CpuOracle(A, mu, c), _gpu(A, mu, c)
        cc, gc = cpu.make_cache(x), gpu.make_cache(x)
        _close(gpu.value(gc), cpu.value(cc))
        z = A @ x
        _close(gpu.gradient(gc), cpu.gradient(cc),
               _absscale(A, (2 * c[1] * z - 3 * c[2] * z * z + 4 * c[3] * z ** 3) / T))
        H = gpu.hvp(gc, V)
        psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
        for i in range(4):
            _close(H[i], cpu.hvp(cc, V[i]), _absscale(A, psi2 * (A @ V[i]) / T))


def test_device_path_matches_host_path():
    torch = pytest.importorskip("torch")
    from paper_2604_25378_b200.datagen import make_panel, random_simplex_point, random_tangents
    A, mu, c = make_panel("C2", seed=2)
    T, n = A.shape
    Xd = torch.from_numpy(A).cuda()
    gpu = _gpu(None, mu, c, device_panel=(Xd.data_ptr(), n, T, n))
    host = _gpu(A, mu, c)
    x = random_simplex_point(n, 1)
    V = random_tangents(n, 8, 1)
    xd = torch.from_numpy(x).cuda()
    Vd = torch.from_numpy(V).cuda()
    out = torch.empty_like(Vd)
    gpu.make_cache_device(0, xd.data_ptr())
    gpu.hvp_device(0, Vd.data_ptr(), 8, out.data_ptr())
    sums = torch.empty(9, dtype=torch.float64, device="cuda")
    gpu.line_sums_device(0, Vd[0].data_ptr(), sums.data_ptr())
    gpu.synchronize()
    hc = host.make_cache(x)
    np.testing.assert_array_equal(out.cpu().numpy(), host.hvp(hc, V))
    lm = host.line_model(hc, V[0], 1.0)
    np.testing.assert_array_equal(sums.cpu().numpy(), lm.sums)
    z, g, s = gpu.slot_pointers(0)
    assert z and g and s


def test_nccl_single_rank_group_path():
    """With an NCCL unique id the context builds a communicator (here a 1-rank
    group) and every op runs the multi-GPU finish path: fixed-order partial
    reduction -> ncclAllReduce(sum, fp64) -> epilogue. Results must equal the
    single-GPU path bit for bit (an allreduce over one rank is a copy)."""
    from paper_2604_25378_b200.gpu_oracle import nccl_unique_id
    A, mu = rh.lcg_panel(64, 777, 5)
    c = rh.crra(10.0)
    T = A.shape[0]
    plain = _gpu(A, mu, c)
    group = _gpu(A, mu, c, rank=0, nranks=1, row0=0, T_global=T, nccl_id=nccl_unique_id())
    x = rh.simplex_point(64, 3)
    V = np.random.default_rng(1).standard_normal((8, 64))
    cp, cg = plain.make_cache(x), group.make_cache(x)
    assert plain.value(cp) == group.value(cg)
    np.testing.assert_array_equal(plain.gradient(cp), group.gradient(cg))
    np.testing.assert_array_equal(plain.hvp(cp, V), group.hvp(cg, V))
    np.testing.assert_array_equal(plain.third_action(cp, V[:3], V[3:6]), group.third_action(cg, V[:3], V[3:6]))
    d = V[0] - V[0].mean()
    lp, lg = plain.line_model(cp, d, 1.0), group.line_model(cg, d, 1.0)
    np.testing.assert_array_equal(lp.sums, lg.sums)
    np.testing.assert_array_equal(plain.weighted_gram(cp), group.weighted_gram(cg))
    from paper_2604_25378_b200.gpu_oracle import preset
    xs1, r1 = plain.solve(preset("large"))
    xs2, r2 = group.solve(preset("large"))
    np.testing.assert_array_equal(xs1, xs2)


def test_binary_ingest_matches_host_centering(tmp_path):
    """mvsk_gpu_create_from_binary: raw returns file -> device rows -> centred
    on the device; oracle outputs match the CPU oracle on the host-centred panel,
    and a non-finite entry raises DataError (center_panel, panel.hpp:38-39)."""
    from paper_2604_25378_b200.gpu_oracle import DataError, GpuOracle, save_returns_binary
    R = rh.lcg_panel_raw(37, 400, 8)
    path = tmp_path / "panel.bin"
    save_returns_binary(path, R)
    c = rh.crra(10.0)
    g = GpuOracle.from_binary(path, c)
    A, mu = po.center_panel(R)
    np.testing.assert_allclose(g.mu, mu, rtol=1e-14, atol=1e-17)
    cpu = po.CpuOracle(A, mu, c)
    x = rh.simplex_point(37, 5)
    gc, cc = g.make_cache(x), cpu.make_cache(x)
    assert abs(g.value(gc) - cpu.value(cc)) <= 1e-12 * (1 + abs(cpu.value(cc)))
    np.testing.assert_allclose(g.gradient(gc), cpu.gradient(cc), rtol=1e-10, atol=1e-13)
    R[3, 4] = np.nan
    save_returns_binary(path, R)
    with pytest.raises(DataError):
        GpuOracle.from_binary(path, c)


@pytest.mark.parametrize("n,T", [(8192, 64), (8190, 3), (2, 2), (3, 1000), (1, 2)])
def test_edge_shapes(n, T):
    """Widest supported rows (n = 8192), odd n, the minimum T = 2, a tall-thin
    panel and n = 1: parity with the CPU oracle for f, g and a 3-RHS HVP."""
    rng = np.random.default_rng(n * 7 + T)
    A = rng.uniform(-0.1, 0.4, (T, n))
    A -= A.mean(axis=0)
    mu = rng.uniform(0, 5e-4, n)
    c = rh.crra(10.0)
    x = rng.exponential(size=n)
    x /= x.sum()
    V = rng.standard_normal((3, n))
    cpu, gpu = po.CpuOracle(A, mu, c), _gpu(A, mu, c)
    cc, gc = cpu.make_cache(x), gpu.make_cache(x)
    _close(gpu.value(gc), cpu.value(cc))
    z = A @ x
    _close(gpu.gradient(gc), cpu.gradient(cc), _absscale(A, (2 * c[1] * z - 3 * c[2] * z * z + 4 * c[3] * z ** 3) / T))
    H = gpu.hvp(gc, V)
    psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
    for i in range(3):
        _close(H[i], cpu.hvp(cc, V[i]), _absscale(A, psi2 * (A @ V[i]) / T))


def test_contract_violations():
    """Typed errors at the boundary: too-wide rows, RHS count, slots, faces."""
    from paper_2604_25378_b200.gpu_oracle import DimensionError, DomainError
    A, mu = rh.lcg_panel(6, 20, 3)
    g = _gpu(A, mu, rh.crra(4.0))
    cache = g.make_cache(rh.simplex_point(6, 1))
    with pytest.raises(DimensionError):
        g.hvp(cache, np.ones((17, 6)))  # > MVSK_GPU_MAX_RHS
    with pytest.raises(DomainError):
        g.make_cache(rh.simplex_point(6, 1), slot=8)
    with pytest.raises(DomainError):
        g.set_face(np.array([3, 1]), 1e-8)  # not increasing
    with pytest.raises(DomainError):
        g.set_face(np.array([], dtype=np.int64), 1e-8)  # degenerate face
    g.set_face(np.array([0, 2, 5]), 1e-8)
    with pytest.raises(DomainError):  # slots were invalidated by the face change
        g.gradient(cache)
    wide = np.zeros((2, 8200))
    with pytest.raises(DimensionError):
        gw = _gpu(wide, np.zeros(8200), rh.crra(2.0))
        gw.make_cache(np.full(8200, 1 / 8200))
    H16 = g.hvp(g.make_cache(np.array([0.4, 0.3, 0.3])), np.ones((16, 3)) * np.array([1.0, -1.0, 0.0]))
    assert H16.shape == (16, 3) and np.all(H16 == H16[0])


def test_graph_replay_tracks_inputs_and_offsets():
    """Host-API ops are replayed as CUDA graphs from their third call on
    (host_ops.cu run_graphed). Every replay must see the new inputs, and a
    set_offset (which moves/changes buffers baked into the graph) must
    invalidate the captured graphs."""
    A, mu = rh.lcg_panel(24, 300, 17)
    c = rh.crra(8.0)
    T, n = A.shape
    cpu = po.CpuOracle(A, mu, c)
    gpu = _gpu(A, mu, c)
    rng = np.random.default_rng(3)
    for it in range(6):
        x = rng.dirichlet(np.ones(n))
        gc, cc = gpu.make_cache(x), cpu.make_cache(x)
        assert abs(gpu.value(gc) - cpu.value(cc)) <= 1e-12 * (1 + abs(cpu.value(cc)))
        _close(gpu.gradient(gc), cpu.gradient(cc))
        V = rng.standard_normal((3, n))
        H = gpu.hvp(gc, V)
        for i in range(3):
            _close(H[i], cpu.hvp(cc, V[i]))
        d = rng.standard_normal(n)
        d -= d.mean()
        cap = po.alpha_max(x, d, 0.0)
        mg, mc = gpu.line_model(gc, d, cap), cpu.line_model(cc, d, cap)
        got = np.array([mg.a0, mg.a1, mg.a2, mg.a3, mg.a4, *mg.sums])
        np.testing.assert_allclose(got, mc, rtol=1e-11, atol=1e-14 * np.max(np.abs(mc)))
    zoff = rng.standard_normal(T) * 1e-3
    for it in range(4):
        gpu.set_offset(zoff * (it + 1), 1e-4 * it)
        off = po.CpuOracle(A, mu, c, zoff=zoff * (it + 1), value_offset=1e-4 * it)
        x = rng.dirichlet(np.ones(n))
        gc, cc = gpu.make_cache(x), off.make_cache(x)
        assert abs(gpu.value(gc) - off.value(cc)) <= 1e-12 * (1 + abs(off.value(cc)))
        _close(gpu.gradient(gc), off.gradient(cc))
        v = rng.standard_normal(n)
        _close(gpu.hvp(gc, v), off.hvp(cc, v))
    assert gpu.passes()[2] > 0
    gpu.close()


def test_set_coeffs_and_sweep_contract():
    """set_coeffs replaces c on a live context (cached slots invalidated, f and
    g follow the new coefficients); the floor sweep rejects bad arguments and
    restores the context's coefficients."""
    from paper_2604_25378_b200.gpu_oracle import DomainError, preset
    A, mu = rh.lcg_panel(7, 60, 12)
    c1, c2 = rh.crra(4.0), rh.crra(9.0)
    g = _gpu(A, mu, c1)
    x = rh.simplex_point(7, 2)
    cache = g.make_cache(x)
    g.set_coeffs(c2)
    with pytest.raises(DomainError):
        g.gradient(cache)  # invalidated
    cpu = po.CpuOracle(A, mu, c2)
    cc = cpu.make_cache(x)
    gc = g.make_cache(x)
    assert abs(g.value(gc) - cpu.value(cc)) <= 1e-12 * (1 + abs(cpu.value(cc)))
    _close(g.gradient(gc), cpu.gradient(cc))
    with pytest.raises(DomainError):
        g.set_coeffs([np.nan, 1.0, 1.0, 1.0])
    cfg = preset("small")
    cfg.has_max_elapsed = 0
    with pytest.raises(DomainError):
        g.floor_sweep(cfg, floors=[0.1, np.inf])
    with pytest.raises(DomainError):
        g.floor_sweep(cfg, nfloors=0)
    out = g.floor_sweep(cfg, floors=[float(mu.mean())], max_solves=6)
    assert len(out.points) == 1 and out.total_solves >= 2
    gc2 = g.make_cache(x)  # coefficients restored to c2
    assert abs(g.value(gc2) - cpu.value(cc)) <= 1e-12 * (1 + abs(cpu.value(cc)))
