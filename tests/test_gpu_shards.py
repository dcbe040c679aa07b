"""Row-sharded execution checked on ONE GPU.

The driver's boxes have one GPU, and NCCL refuses two ranks on one device, so
the N > 1 code paths are exercised through the in-process group
(mvsk_gpu_group, collective.cu): nranks contexts, each owning a contiguous row
block, driven SPMD by one host thread per rank, whose exchange step is a
peer-memory allreduce instead of ncclAllReduce. Everything else is the
production N > 1 path: passes with the split finish (do_epi = 0), the
allreduce of the n-vector / power sums, the packed n (n + 1) / 2 Gram
exchange, the cluster-resident kernels switched off (nranks > 1), the
replicated host driver. Bars (written per check):
* every rank holds bitwise identical results;
* sharded vs one context: oracle values to 1e-13 relative (only the
  summation split differs), solves same status / active set, weights 1e-8;
* sharded vs the CPU parity oracle: 1e-11 relative (north_star).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import pyoracle as po
from tests import refhelpers as rh

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), 1e-300)


def _shards(A, mu, c, nranks):
    from paper_2604_25378_b200.gpu_oracle import GpuGroup, GpuOracle
    T = A.shape[0]
    grp = GpuGroup(nranks)
    b = [T * r // nranks for r in range(nranks + 1)]
    members = [GpuOracle(A[b[r]:b[r + 1]], mu, c, row0=b[r], T_global=T, group=grp, rank=r) for r in range(nranks)]
    return grp, members, b


def _spmd(members, fn):
    with ThreadPoolExecutor(len(members)) as ex:
        return list(ex.map(lambda r: fn(members[r], r), range(len(members))))


def _close(grp, members):
    for m in members:
        m.close()
    grp.close()


@pytest.mark.parametrize("name,nranks", [("C1", 2), ("C2", 2), ("C2", 3), ("C3", 2)])
def test_sharded_oracle_ops_match_single_context_and_oracle(name, nranks):
    from paper_2604_25378_b200.datagen import make_panel, random_simplex_point, random_tangents
    from paper_2604_25378_b200.gpu_oracle import GpuOracle
    A, mu, c = make_panel(name, seed=21, kappa=100.0 if name == "C2" else None)
    T, n = A.shape
    x = random_simplex_point(n, 3)
    V = random_tangents(n, 8, 4)
    U = random_tangents(n, 8, 5)

    def ops(g, r):
        cc = g.make_cache(x)
        out = {"f": g.value(cc), "mom": np.array(g.moments(cc)), "g": g.gradient(cc), "H1": g.hvp(cc, V[:1]),
               "H8": g.hvp(cc, V), "T1": g.third_action(cc, U[:1], V[:1]), "T8": g.third_action(cc, U, V),
               "psi2": g.hessian_diag_weights(cc), "Ad": g.sample_direction(V[0])}
        lm = g.line_model(cc, V[0], 0.05)
        out["lm"] = np.array([lm.a0, lm.a1, lm.a2, lm.a3, lm.a4, *lm.sums])
        out["G"] = g.weighted_gram(cc)
        out["passes"] = g.passes()
        return out

    grp, members, b = _shards(A, mu, c, nranks)
    try:
        res = _spmd(members, ops)
    finally:
        _close(grp, members)
    one = GpuOracle(A, mu, c)
    ref1 = ops(one, 0)
    one.close()
    cpu = po.CpuOracle(A, mu, c)
    cc = cpu.make_cache(x)
    global_keys = ("f", "mom", "g", "H1", "H8", "T1", "T8", "lm", "G")
    # 1. identical bits on every rank
    for r in range(1, nranks):
        for k in global_keys:
            np.testing.assert_array_equal(res[r][k], res[0][k], err_msg=k)
    # 2. local row results concatenate to the full-panel ones
    np.testing.assert_array_equal(np.concatenate([res[r]["psi2"] for r in range(nranks)]), ref1["psi2"])
    assert _rel(np.concatenate([res[r]["Ad"] for r in range(nranks)]), ref1["Ad"]) <= 1e-13
    # 3. vs one context: 1e-13 relative (summation split only)
    s = res[0]
    for k in global_keys:
        assert _rel(s[k], ref1[k]) <= 1e-13, (k, _rel(s[k], ref1[k]))
    assert s["passes"] == ref1["passes"]
    # 4. vs the CPU parity oracle: 1e-11 relative (north_star)
    assert abs(s["f"] - cpu.value(cc)) <= 1e-11 * abs(cpu.value(cc))
    assert _rel(s["g"], cpu.gradient(cc)) <= 1e-11
    for i in range(8):
        assert _rel(s["H8"][i], cpu.hvp(cc, V[i])) <= 1e-11
        assert _rel(s["T8"][i], cpu.third_action(cc, U[i], V[i])) <= 1e-11
    assert _rel(s["lm"], cpu.line_model(cc, V[0], 0.05)) <= 1e-11
    psi2 = cpu.hessian_diag_weights(cc)
    G_ref = (A * psi2[:, None]).T @ A / T
    assert _rel(s["G"], G_ref) <= 1e-11
    np.testing.assert_array_equal(s["G"], s["G"].T)


@pytest.mark.parametrize("name,preset", [("C1", "small"), ("C2", "large"), ("C3", "large")])
def test_sharded_solve_is_replicated_and_matches(name, preset):
    """solve (solver.hpp:195-655) as an SPMD-replicated driver over 2 shards:
    both ranks end on identical bits, equal to the one-context solve and the
    reference-exact CPU oracle at the north_star bar."""
    from paper_2604_25378_b200.datagen import crra, make_panel
    from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset as gpreset
    A, mu, c = make_panel(name, seed=22)
    if name == "C3":
        c = crra(5.0)
    cfg = gpreset(preset)
    cfg.has_max_elapsed = 0
    cfg.epsilon = 1e-10
    grp, members, _ = _shards(A, mu, c, 2)
    try:
        res = _spmd(members, lambda g, r: g.solve(cfg))
    finally:
        _close(grp, members)
    (x0, r0), (x1, r1) = res
    np.testing.assert_array_equal(x0, x1)
    assert (r0.status, r0.iterations, r0.f_star) == (r1.status, r1.iterations, r1.f_star)
    one = GpuOracle(A, mu, c)
    xs, rs = one.solve(cfg)
    one.close()
    ccfg = po.preset(preset)
    ccfg.has_max_elapsed = 0
    ccfg.epsilon = 1e-10
    xc, rc = po.solve(A, mu, c, ccfg)
    for xo, ro in ((xs, rs), (xc, rc)):
        assert r0.status == ro.status
        act = lambda v: tuple(np.nonzero(v <= cfg.tau + 1e-12)[0])  # noqa: E731
        assert act(x0) == act(xo)
        assert abs(r0.f_star - ro.f_star) <= 1e-12 * (1 + abs(ro.f_star))
        assert float(np.max(np.abs(x0 - xo))) <= 1e-8


def test_group_lifecycle_errors():
    from paper_2604_25378_b200.gpu_oracle import DomainError, GpuGroup
    with pytest.raises(DomainError):
        GpuGroup(0)
    with pytest.raises(DomainError):
        GpuGroup(9)
    A, mu = rh.lcg_panel(4, 20, 1)
    grp, members, _ = _shards(A, mu, rh.crra(3.0), 2)
    with pytest.raises(DomainError):
        grp.close()  # members alive
    _close(grp, members)
