"""Multi-rank host logic on CPU (gloo, world_size 2): the row sharding the
multi-GPU path uses: shard_rows partitions T, each rank
generates exactly its rows of the panel, the global centring mean is an
allreduce of column sums, and every oracle output is a sum over samples, so
per-shard partials + allreduce reproduce the single-rank oracle and every rank
receives bitwise-identical results (the SPMD driver stays in lock-step)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_25378_b200.datagen import CONFIGS, crra, raw_returns
from paper_2604_25378_b200.gpu_oracle import shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    spec = CONFIGS["C2"]
    T, n = spec.T, spec.n
    row0, T_loc = shard_rows(T, ws, rank)
    R = raw_returns(spec, 3, rows=(row0, row0 + T_loc))
    colsum = R.sum(dim=0)
    dist.all_reduce(colsum)
    mu = colsum / T
    A = (R - mu).numpy()
    c = crra(spec.gamma)
    x = np.full(n, 1.0 / n)
    v = np.linspace(-1, 1, n)
    v -= v.mean()
    z = A @ x
    w = (2 * c[1] * z - 3 * c[2] * z * z + 4 * c[3] * z ** 3) / T
    psi2 = 2 * c[1] - 6 * c[2] * z + 12 * c[3] * z * z
    part = np.concatenate([A.T @ w, A.T @ (psi2 * (A @ v) / T),
                           [np.sum(z * z), np.sum(z ** 3), np.sum(z ** 4)]])
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    q.put((rank, row0, T_loc, mu.numpy(), t.numpy()))
    dist.destroy_process_group()


def test_row_shard_partition():
    for T in (1, 7, 500, 262144):
        for ws in (1, 2, 3, 8):
            blocks = [shard_rows(T, ws, r) for r in range(ws)]
            assert blocks[0][0] == 0
            for (a, na), (b, _) in zip(blocks, blocks[1:]):
                assert a + na == b
            assert blocks[-1][0] + blocks[-1][1] == T
            assert max(b[1] for b in blocks) - min(b[1] for b in blocks) <= 1


def test_sharded_rows_are_bitwise_rows_of_the_full_panel():
    spec = CONFIGS["C1"]
    full = raw_returns(spec, 9)
    for lo, hi in ((0, 17), (17, 333), (250, 500)):
        assert torch.equal(raw_returns(spec, 9, rows=(lo, hi)), full[lo:hi])


def test_gloo_two_rank_oracle_reduction():
    from oracle import pyoracle as po
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, _, _, mu0, t0), (_, _, _, mu1, t1) = res
    assert np.array_equal(t0, t1) and np.array_equal(mu0, mu1)  # identical on every rank
    spec = CONFIGS["C2"]
    R = raw_returns(spec, 3).numpy()
    mu = R.sum(axis=0) / spec.T
    A = R - mu
    np.testing.assert_allclose(mu0, mu, rtol=1e-13, atol=1e-18)
    c = crra(spec.gamma)
    n = spec.n
    o = po.CpuOracle(A, mu, c)
    x = np.full(n, 1.0 / n)
    v = np.linspace(-1, 1, n)
    v -= v.mean()
    cache = o.make_cache(x)
    g_ref = o.gradient(cache)
    g = -c[0] * mu + t0[:n]
    assert np.max(np.abs(g - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))
    h_ref = o.hvp(cache, v)
    assert np.max(np.abs(t0[n:2 * n] - h_ref)) <= 1e-11 * np.max(np.abs(h_ref))
    m = o.moments(cache)
    np.testing.assert_allclose(t0[2 * n:] / spec.T, m[1:], rtol=1e-12)
