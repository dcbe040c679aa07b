"""Python mirror of the reference operator API over the C-ABI.

``GpuOracle`` has the method set of ``mvsk::Oracle`` (oracle.hpp:29-149);
``OracleCache`` handles are device slots. ``line_model`` mirrors
linesearch.hpp:62-81, ``yand_direction`` affine_normal.hpp:127-245 and
``solve`` solver.hpp:195-655. Typed errors follow common.hpp:14-25. Every call
goes through libmvsk_b200.so (sm_100a); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import (OBSERVER_FN, mvsk_coeffs, mvsk_direction_diag, mvsk_floor_point, mvsk_solve_report,
                   mvsk_solver_config, mvsk_sweep_config,
                   mvsk_tangent_config)


class MvskError(Exception):
    code = 7
    kind = "internal_error"


class DimensionError(MvskError, ValueError):  # mvsk::dimension_error (std::invalid_argument)
    code, kind = 1, "dimension_error"


class DomainError(MvskError, ValueError):  # mvsk::domain_error (std::invalid_argument)
    code, kind = 2, "domain_error"


class DataError(MvskError, RuntimeError):
    code, kind = 3, "data_error"


class NumericError(MvskError, RuntimeError):
    code, kind = 4, "numeric_error"


class CudaError(MvskError, RuntimeError):
    code, kind = 5, "cuda_error"


class NcclError(MvskError, RuntimeError):
    code, kind = 6, "nccl_error"


_ERR = {1: DimensionError, 2: DomainError, 3: DataError, 4: NumericError, 5: CudaError, 6: NcclError}

_D = C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data_as(_D)


def _vec(a, n=None):
    x = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and x.shape[-1] != n:
        raise DimensionError(f"vector length {x.shape[-1]} does not match {n}")
    return x


def _raise(lib, ctx, code):
    if code == 0:
        return
    msg = lib.mvsk_gpu_last_error(ctx).decode() if ctx is not None else "error"
    raise _ERR.get(code, MvskError)(msg)


def crra_coefficients(gamma: float) -> np.ndarray:
    """panel.hpp:76-87"""
    if not gamma > 0:
        raise DomainError("crra_coefficients: gamma must be positive")
    g = float(gamma)
    return np.array([1.0, g / 2.0, g * (g + 1.0) / 6.0, g * (g + 1.0) * (g + 2.0) / 24.0])


def center_panel(R: np.ndarray):
    """panel.hpp:32-44: returns (A, mu)."""
    R = np.asarray(R, dtype=np.float64)
    if R.shape[0] < 2:
        raise DimensionError("center_panel: need at least two time periods")
    if R.shape[1] < 1:
        raise DimensionError("center_panel: need at least one asset")
    if not np.all(np.isfinite(R)):
        raise DataError("center_panel: non-finite return entry")
    mu = R.sum(axis=0) / R.shape[0]
    return R - mu[None, :], mu


class OracleCache:
    """Device-resident cache (a slot of the context)."""

    def __init__(self, oracle: "GpuOracle", slot: int, f: float):
        self.oracle = oracle
        self.slot = slot
        self.f_value = f


@dataclass
class LineModel:
    a0: float
    a1: float
    a2: float
    a3: float
    a4: float
    alpha_cap: float
    sums: np.ndarray

    def eval(self, alpha):
        return self.a0 + alpha * (self.a1 + alpha * (self.a2 + alpha * (self.a3 + alpha * self.a4)))


@dataclass
class FloorSweep:
    """Result of GpuOracle.floor_sweep: one calibrated optimum per return floor."""
    points: list  # of dicts: floor, c1, mean, f_star, kkt_residual, status, solves
    X: np.ndarray  # nfloors x n optima
    m_mv: float  # in-sample mean of the minimum-variance optimum
    m_max: float  # max_j mu_j (max-mean vertex)
    total_solves: int


class GpuGroup:
    """In-process row-shard group (mvsk_gpu_group): nranks GpuOracle shards in
    this process, one host thread per rank, combined by the peer-memory
    allreduce of collective.cu instead of NCCL. Close the members first."""

    def __init__(self, nranks: int):
        self.lib = _abi.load_library()
        self._g = C.c_void_p()
        code = self.lib.mvsk_gpu_group_create(int(nranks), C.byref(self._g))
        if code != 0:
            raise _ERR.get(code, MvskError)(self.lib.mvsk_gpu_last_error(None).decode())
        self.nranks = int(nranks)

    def close(self):
        if self._g and self._g.value:
            code = self.lib.mvsk_gpu_group_destroy(self._g)
            if code != 0:
                raise _ERR.get(code, MvskError)(self.lib.mvsk_gpu_last_error(None).decode())
            self._g = C.c_void_p()


class GpuOracle:
    """mvsk::Oracle over a panel resident in B200 HBM (or a row shard of it)."""

    def __init__(self, A, mu, coeffs, device: int = 0, *, rank: int = 0, nranks: int = 1, row0: int = 0,
                 T_global: int | None = None, nccl_id: bytes | None = None, device_panel=None,
                 group: "GpuGroup | None" = None):
        self.lib = _abi.load_library()
        self._ctx = C.c_void_p()
        self.c = _vec(coeffs, 4)
        cf = mvsk_coeffs(*self.c)
        if device_panel is not None:
            # borrowed device memory (e.g. a torch CUDA tensor): (ptr, ld, T_local, n)
            ptr, ld, T_local, n = device_panel
            self.mu = _vec(mu, n)
            self.n = n
            self.T_local = T_local
            self.T = T_global if T_global is not None else T_local
            idb = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            code = self.lib.mvsk_gpu_create_from_device(C.c_void_p(ptr), ld, T_local, row0, self.T, n, _p(self.mu),
                                                        C.byref(cf), device, nranks, rank, idb, C.byref(self._ctx))
        else:
            A = np.ascontiguousarray(A, dtype=np.float64)
            if A.ndim != 2:
                raise DimensionError("panel must be 2-D")
            self.T_local, self.n = A.shape
            self.T = T_global if T_global is not None else self.T_local
            if np.asarray(mu).size != self.n:
                raise DimensionError("oracle: mu length does not match panel columns")
            self.mu = _vec(mu, self.n)
            idb = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            if group is not None:
                code = self.lib.mvsk_gpu_create_sharded_in_group(_p(A), self.T_local, row0, self.T, self.n,
                                                                 _p(self.mu), C.byref(cf), device, group._g, rank,
                                                                 C.byref(self._ctx))
            else:
                code = self.lib.mvsk_gpu_create_sharded(_p(A), self.T_local, row0, self.T, self.n, _p(self.mu),
                                                        C.byref(cf), device, nranks, rank, idb, C.byref(self._ctx))
        if code != 0:
            raise _ERR.get(code, MvskError)(self.lib.mvsk_gpu_last_error(None).decode())
        self._m = self.n
        self._next_slot = 0

    @classmethod
    def from_binary(cls, path, coeffs, device: int = 0, *, rank: int = 0, nranks: int = 1,
                    nccl_id: bytes | None = None) -> "GpuOracle":
        """load_returns_binary + center_panel + Oracle (panel_io.hpp:121-141):
        this rank's rows of a binary panel file go straight to device memory."""
        self = cls.__new__(cls)
        self.lib = _abi.load_library()
        self._ctx = C.c_void_p()
        self.c = _vec(coeffs, 4)
        cf = mvsk_coeffs(*self.c)
        idb = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        code = self.lib.mvsk_gpu_create_from_binary(str(path).encode(), C.byref(cf), device, nranks, rank, idb,
                                                    C.byref(self._ctx))
        if code != 0:
            raise _ERR.get(code, MvskError)(self.lib.mvsk_gpu_last_error(None).decode())
        Tg, Tl, n = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.mvsk_gpu_dims(self._ctx, C.byref(Tg), C.byref(Tl), C.byref(n))
        self.T, self.T_local, self.n = Tg.value, Tl.value, n.value
        self.mu = np.empty(self.n)
        self.lib.mvsk_gpu_mu(self._ctx, _p(self.mu))
        self._m = self.n
        self._next_slot = 0
        return self

    # ---- lifecycle --------------------------------------------------------
    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self.lib.mvsk_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, code):
        _raise(self.lib, self._ctx, code)

    @property
    def ctx(self):
        return self._ctx

    def set_stream(self, stream_ptr: int | None):
        self._chk(self.lib.mvsk_gpu_set_stream(self._ctx, C.c_void_p(stream_ptr or 0)))

    def synchronize(self):
        self._chk(self.lib.mvsk_gpu_synchronize(self._ctx))

    def periods(self):
        return self.T

    def assets(self):
        return self.n

    # ---- oracle.hpp -------------------------------------------------------
    def set_offset(self, zoff=None, value_offset: float = 0.0):
        z = None if zoff is None else _vec(zoff, self.T_local)
        self._chk(self.lib.mvsk_gpu_set_offset(self._ctx, _p(z), C.c_double(value_offset)))

    def set_face(self, free_idx=None, tau: float = 0.0):
        if free_idx is None:
            self._chk(self.lib.mvsk_gpu_set_face(self._ctx, None, self.n, C.c_double(tau)))
            self._m = self.n
        else:
            idx = np.ascontiguousarray(free_idx, dtype=np.int64)
            self._chk(self.lib.mvsk_gpu_set_face(self._ctx, idx.ctypes.data_as(C.POINTER(C.c_int64)), idx.size,
                                                 C.c_double(tau)))
            self._m = idx.size

    def make_cache(self, x, slot: int | None = None) -> OracleCache:
        x = _vec(x)
        if x.size != self._m:
            raise DimensionError("oracle: iterate length does not match panel")
        if slot is None:
            slot = self._next_slot
            self._next_slot = (self._next_slot + 1) % _abi.MVSK_GPU_MAX_SLOTS
        f = C.c_double()
        self._chk(self.lib.mvsk_gpu_make_cache(self._ctx, slot, _p(x), C.byref(f)))
        return OracleCache(self, slot, f.value)

    def value(self, cache: OracleCache) -> float:
        return cache.f_value

    def moments(self, cache: OracleCache):
        out = np.empty(4)
        self._chk(self.lib.mvsk_gpu_moments(self._ctx, cache.slot, _p(out)))
        return tuple(out)

    def gradient(self, cache: OracleCache) -> np.ndarray:
        g = np.empty(self._m)
        self._chk(self.lib.mvsk_gpu_gradient(self._ctx, cache.slot, _p(g)))
        return g

    def hvp(self, cache: OracleCache, v) -> np.ndarray:
        V = _vec(v, self._m)
        k = 1 if V.ndim == 1 else V.shape[0]
        out = np.empty((k, self._m))
        self._chk(self.lib.mvsk_gpu_hvp(self._ctx, cache.slot, _p(V), k, _p(out)))
        return out[0] if V.ndim == 1 else out

    def third_action(self, cache: OracleCache, u, v) -> np.ndarray:
        U, V = _vec(u, self._m), _vec(v, self._m)
        k = 1 if U.ndim == 1 else U.shape[0]
        out = np.empty((k, self._m))
        self._chk(self.lib.mvsk_gpu_third_action(self._ctx, cache.slot, _p(U), _p(V), k, _p(out)))
        return out[0] if U.ndim == 1 else out

    def hessian_diag_weights(self, cache: OracleCache) -> np.ndarray:
        out = np.empty(self.T_local)
        self._chk(self.lib.mvsk_gpu_hessian_diag_weights(self._ctx, cache.slot, _p(out)))
        return out

    def sample_direction(self, d) -> np.ndarray:
        d = _vec(d, self._m)
        out = np.empty(self.T_local)
        self._chk(self.lib.mvsk_gpu_sample_direction(self._ctx, _p(d), _p(out)))
        return out

    def weighted_gram(self, cache: OracleCache) -> np.ndarray:
        G = np.empty((self._m, self._m))
        self._chk(self.lib.mvsk_gpu_weighted_gram(self._ctx, cache.slot, _p(G)))
        return G

    def passes(self):
        f, t, p = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.mvsk_gpu_passes(self._ctx, C.byref(f), C.byref(t), C.byref(p))
        return f.value, t.value, p.value

    def reset_passes(self):
        self.lib.mvsk_gpu_reset_passes(self._ctx)

    def launch_count(self) -> int:
        """Kernels this context has enqueued (graph replays included)."""
        v = C.c_uint64()
        self._chk(self.lib.mvsk_gpu_launch_count(self._ctx, C.byref(v)))
        return v.value

    # ---- linesearch.hpp / affine_normal.hpp / solver.hpp ------------------
    def line_model(self, cache: OracleCache, d, cap: float) -> LineModel:
        d = _vec(d, self._m)
        out = np.empty(14)
        self._chk(self.lib.mvsk_gpu_line_model(self._ctx, cache.slot, _p(d), C.c_double(cap), _p(out)))
        return LineModel(*out[:5], cap, out[5:].copy())

    def line_models(self, cache: OracleCache, D, caps):
        """k line models in one round trip (mvsk_gpu_line_models): D is k x m; a
        rejected direction comes back with a0 = NaN instead of raising."""
        D = np.ascontiguousarray(np.asarray(D, dtype=np.float64))
        if D.ndim != 2 or D.shape[1] != self._m:
            raise DimensionError("line_models: D must be k x m")
        k = D.shape[0]
        out = np.empty((k, 14))
        self._chk(self.lib.mvsk_gpu_line_models(self._ctx, cache.slot, _p(D), k, _p(out)))
        return [LineModel(*out[i, :5], float(caps[i]), out[i, 5:].copy()) for i in range(k)]

    def yand_direction(self, cache: OracleCache, cfg: mvsk_tangent_config, it_seed: int = 0):
        d = np.empty(self._m)
        diag = mvsk_direction_diag()
        self._chk(self.lib.mvsk_gpu_yand_direction(self._ctx, cache.slot, C.byref(cfg), C.c_uint64(it_seed), _p(d),
                                                   C.byref(diag)))
        return d, diag

    def solve(self, cfg: mvsk_solver_config, x0=None, observer=None):
        xs = np.empty(self.n)
        rep = mvsk_solve_report()
        x0a = None if x0 is None else _vec(x0)
        if x0a is not None and x0a.size != self.n:
            raise DomainError("solve: x0 is not in the tau-slice")
        if observer is not None:
            cb = OBSERVER_FN(lambda _u, it, f, xp, nn: observer(int(it), float(f),
                                                               np.ctypeslib.as_array(xp, (nn,)).copy()))
        else:
            cb = OBSERVER_FN()
        self._chk(self.lib.mvsk_gpu_solve(self._ctx, C.byref(cfg), _p(x0a), _p(xs), C.byref(rep), cb, None))
        return xs, rep

    def set_coeffs(self, coeffs):
        """Replace c1..c4 on the live context (the panel stays resident)."""
        self.c = _vec(coeffs, 4)
        self._chk(self.lib.mvsk_gpu_set_coeffs(self._ctx, C.byref(mvsk_coeffs(*self.c))))

    def floor_sweep(self, cfg: mvsk_solver_config, nfloors: int = 5, floors=None, mean_tol: float = 1e-3,
                    max_solves: int = 16, warm_start: bool = True) -> FloorSweep:
        """Return-floor sweep (BASELINE config 4; c1 calibration of PAPER.md:757,
        not part of the reference code): for each floor, the c1 >= 0 whose
        optimum's in-sample mean is closest to it, c2..c4 fixed."""
        fl = None if floors is None else _vec(floors)
        if fl is not None:
            nfloors = fl.size
        X = np.empty((nfloors, self.n))
        pts = (mvsk_floor_point * nfloors)()
        sw = mvsk_sweep_config(mean_tol, max_solves, 1 if warm_start else 0)
        mmv, mmax, tot = C.c_double(), C.c_double(), C.c_int32()
        self._chk(self.lib.mvsk_gpu_floor_sweep(self._ctx, C.byref(cfg), C.byref(sw), nfloors, _p(fl), _p(X), pts,
                                                C.byref(mmv), C.byref(mmax), C.byref(tot)))
        points = [{k: getattr(p, k) for k, _ in mvsk_floor_point._fields_} for p in pts]
        return FloorSweep(points, X, mmv.value, mmax.value, tot.value)

    # ---- device-resident path (pointers into HBM, async on the context stream)
    def make_cache_device(self, slot: int, x_ptr: int):
        self._chk(self.lib.mvsk_gpu_make_cache_device(self._ctx, slot, C.c_void_p(x_ptr)))

    def hvp_device(self, slot: int, v_ptr: int, k: int, out_ptr: int):
        self._chk(self.lib.mvsk_gpu_hvp_device(self._ctx, slot, C.c_void_p(v_ptr), k, C.c_void_p(out_ptr)))

    def third_action_device(self, slot: int, u_ptr: int, v_ptr: int, k: int, out_ptr: int):
        self._chk(self.lib.mvsk_gpu_third_action_device(self._ctx, slot, C.c_void_p(u_ptr), C.c_void_p(v_ptr), k,
                                                        C.c_void_p(out_ptr)))

    def line_sums_device(self, slot: int, d_ptr: int, out_ptr: int):
        self._chk(self.lib.mvsk_gpu_line_sums_device(self._ctx, slot, C.c_void_p(d_ptr), C.c_void_p(out_ptr)))

    def weighted_gram_device(self, slot: int, G_ptr: int):
        self._chk(self.lib.mvsk_gpu_weighted_gram_device(self._ctx, slot, C.c_void_p(G_ptr)))

    def slot_pointers(self, slot: int):
        z, g, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._chk(self.lib.mvsk_gpu_slot_pointers(self._ctx, slot, C.byref(z), C.byref(g), C.byref(s)))
        return z.value, g.value, s.value


def preset(name: str) -> mvsk_solver_config:
    """small_preset / large_preset (solver.hpp:64-85)."""
    lib = _abi.load_library()
    cfg = mvsk_solver_config()
    code = lib.mvsk_gpu_preset(name.encode(), C.byref(cfg))
    if code != 0:
        raise DomainError(f"preset: unknown mode {name}")
    return cfg


def tangent_config(mode="direct", lam=0.0, krylov_tol=1e-3, krylov_maxit=15, jacobi=False, exact_trace=False,
                   probes=8, probe_maxit=5) -> mvsk_tangent_config:
    """TangentSolveConfig (affine_normal.hpp:59-69)."""
    t = mvsk_tangent_config()
    t.mode = 1 if mode == "pcg" else 0
    t.lambda_ = lam
    t.krylov_tol = krylov_tol
    t.krylov_maxit = krylov_maxit
    t.jacobi = int(jacobi)
    t.exact_trace = int(exact_trace)
    t.hutchinson_probes = probes
    t.probe_maxit = probe_maxit
    return t


def nccl_unique_id() -> bytes:
    lib = _abi.load_library()
    buf = C.create_string_buffer(128)
    code = lib.mvsk_gpu_nccl_unique_id(buf)
    if code != 0:
        raise NcclError(lib.mvsk_gpu_last_error(None).decode())
    return buf.raw


def shard_rows(T: int, nranks: int, rank: int):
    """Contiguous row block of `rank` in a T-row panel split over `nranks`
    (the row-sharding of SURVEY.md §8(e)): [row0, row0 + T_local)."""
    lo = T * rank // nranks
    hi = T * (rank + 1) // nranks
    return lo, hi - lo


def binary_dims(path) -> tuple[int, int]:
    """Header of a binary panel file (panel_io.hpp:123-134): (T, n); raises DataError."""
    lib = _abi.load_library()
    T, n = C.c_int64(), C.c_int64()
    code = lib.mvsk_gpu_binary_dims(str(path).encode(), C.byref(T), C.byref(n))
    if code != 0:
        raise _ERR.get(code, MvskError)(lib.mvsk_gpu_last_error(None).decode())
    return T.value, n.value


def save_returns_binary(path, R: np.ndarray) -> None:
    """Writer of the reference's binary panel format (panel_io.hpp:143-154)."""
    R = np.ascontiguousarray(R, dtype="<f8")
    T, n = R.shape
    with open(path, "wb") as f:
        f.write(b"MVSK")
        f.write(np.array([T, n], dtype="<u4").tobytes())
        f.write(R.tobytes())
