"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU parity oracle.

Two implementations export the same ``mo_*`` surface:

* ``"port"``: ``oracle/_build/libmvsk_oracle.so``, the C++ restatement of the
  reference in ``oracle/mvsk_oracle.{hpp,cpp}`` (no Eigen; runs anywhere);
* ``"reference"``: ``oracle/_ref/libmvsk_ref.so``, the reference's own headers
  (/root/reference/proj/include/mvsk/*.hpp, unmodified) compiled over the Eigen
  API stand-in in ``oracle/ref/`` (built only where /root/reference exists;
  the prebuilt .so travels with the snapshot); ``"reference_native"`` is the
  same code with best-CPU flags, the timed reference arm of bench.py.

This module binds the implementation named by ``MVSK_ORACLE_IMPL`` (default
``port``); ``variant(name)`` returns an independent copy of this module bound
to another one, so a test can hold both side by side. Importable only from
tests/, ``__graft_entry__.smoke()``, the golden-fixture script and bench.py's
CPU legs; the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2604_25378_b200._abi import (OBSERVER_FN, mvsk_direction_diag, mvsk_solve_report,
                                        mvsk_solver_config, mvsk_tangent_config)

ORACLE_DIR = Path(__file__).resolve().parent
REFERENCE_DIR = Path("/root/reference/proj")
LIBS = {
    "port": ORACLE_DIR / "_build" / "libmvsk_oracle.so",
    "reference": ORACLE_DIR / "_ref" / "libmvsk_ref.so",
    "reference_native": ORACLE_DIR / "_ref" / "libmvsk_ref_native.so",
}
IMPL = globals().get("_IMPL_OVERRIDE") or os.environ.get("MVSK_ORACLE_IMPL", "port")
if IMPL not in LIBS:
    raise ValueError(f"MVSK_ORACLE_IMPL={IMPL!r}: expected one of {sorted(LIBS)}")
LIB_PATH = LIBS[IMPL]

ERRORS = {1: "dimension_error", 2: "domain_error", 3: "data_error", 4: "numeric_error", 7: "error"}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "error")


def build() -> Path:
    if IMPL == "port":
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    elif REFERENCE_DIR.exists():
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR / "ref"), f"REF={REFERENCE_DIR}"], check=True)
    else:
        raise FileNotFoundError(f"{LIB_PATH} is not built and {REFERENCE_DIR} is absent")
    return LIB_PATH


def available(impl: str) -> bool:
    """True when `impl`'s library exists or can be built here."""
    return LIBS[impl].exists() or (impl == "port") or REFERENCE_DIR.exists()


_VARIANTS: dict = {}


def variant(impl: str):
    """An independent copy of this module bound to implementation `impl`."""
    if impl == IMPL:
        import sys
        return sys.modules[__name__]
    if impl not in _VARIANTS:
        spec = importlib.util.spec_from_file_location(f"{__name__}__{impl}", __file__)
        mod = importlib.util.module_from_spec(spec)
        mod.__dict__["_IMPL_OVERRIDE"] = impl
        spec.loader.exec_module(mod)
        _VARIANTS[impl] = mod
    return _VARIANTS[impl]


_lib = None
_D = C.POINTER(C.c_double)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.mo_last_error.restype = C.c_char_p
        L.mo_alpha_max.restype = C.c_double
        L.mo_projected_kkt_residual.restype = C.c_double
        L.mo_gradient_mapping_residual.restype = C.c_double
        for name in ("mo_alpha_max",):
            getattr(L, name).argtypes = [_D, _D, C.c_int64, C.c_double]
        L.mo_projected_kkt_residual.argtypes = [_D, C.c_int64]
        L.mo_gradient_mapping_residual.argtypes = [_D, _D, C.c_int64, C.c_double]
        L.mo_splitmix_draw.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_double, C.c_double, C.c_void_p]
        L.mo_set_threads.argtypes = [C.c_int]
        if hasattr(L, "mo_impl"):
            L.mo_impl.restype = C.c_char_p
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _arr(a, n=None) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and x.size != n:
        raise ValueError("length")
    return x


def _check(code: int):
    if code != 0:
        raise OracleError(code, lib().mo_last_error().decode())


def set_threads(t: int):
    lib().mo_set_threads(int(t))


def impl_name() -> str:
    """"reference" for the compiled reference headers, "port" for the restatement."""
    L = lib()
    return L.mo_impl().decode() if hasattr(L, "mo_impl") else "port"


def hvp_throughput(oracle: "CpuOracle", cache: "Cache", V, threads: int, reps: int):
    """Reference arm timing (libmvsk_ref*.so only): `threads` host threads each run
    `reps` reference HVPs over the shared panel and cache. Returns (seconds,
    first result of every thread as a threads x n array)."""
    V = np.ascontiguousarray(V, dtype=np.float64).reshape(-1, oracle.n)
    first = np.empty((threads, oracle.n))
    sec = C.c_double()
    _check(lib().mo_hvp_throughput(oracle.h, cache.h, _p(V), C.c_int(V.shape[0]), C.c_int(threads), C.c_int(reps),
                                   C.byref(sec), _p(first)))
    return sec.value, first


# ---- rng.hpp ---------------------------------------------------------------
def splitmix(seed: int, kind: str, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    k = {"u64": 0, "unit": 1, "normal": 2, "sign": 3, "uniform": 4}[kind]
    out = np.empty(count, dtype=np.uint64 if k == 0 else np.float64)
    lib().mo_splitmix_draw(C.c_uint64(seed), k, count, lo, hi, out.ctypes.data_as(C.c_void_p))
    return out


# ---- panel.hpp -------------------------------------------------------------
def center_panel(R: np.ndarray):
    R = np.ascontiguousarray(R, dtype=np.float64)
    T, n = R.shape
    A = np.empty_like(R)
    mu = np.empty(n)
    _check(lib().mo_center_panel(_p(R), C.c_int64(T), C.c_int64(n), _p(A), _p(mu)))
    return A, mu


def crra(gamma: float) -> np.ndarray:
    out = np.empty(4)
    _check(lib().mo_crra(C.c_double(gamma), _p(out)))
    return out


def make_coefficients(c1, c2, c3, c4) -> np.ndarray:
    out = np.empty(4)
    _check(lib().mo_make_coefficients(*(C.c_double(v) for v in (c1, c2, c3, c4)), _p(out)))
    return out


# ---- oracle.hpp ------------------------------------------------------------
class Cache:
    def __init__(self, oracle: "CpuOracle", handle):
        self._o = oracle
        self.h = handle

    def __del__(self):
        if self.h:
            lib().mo_cache_destroy(self.h)
            self.h = None

    @property
    def z(self) -> np.ndarray:
        out = np.empty(self._o.T)
        lib().mo_cache_z(self.h, _p(out))
        return out


class CpuOracle:
    """Mirror of mvsk::Oracle (oracle.hpp:29-149) over the CPU restatement."""

    def __init__(self, A, mu, coeffs, zoff=None, value_offset: float = 0.0):
        self.A = np.ascontiguousarray(A, dtype=np.float64)
        self.T, self.n = self.A.shape
        self.mu = _arr(mu)
        self.c = _arr(coeffs, 4)
        self._zoff = None if zoff is None else _arr(zoff, self.T)
        h = C.c_void_p()
        _check(lib().mo_oracle_create(_p(self.A), C.c_int64(self.T), C.c_int64(self.n), _p(self.mu),
                                      _p(self.c), _p(self._zoff), C.c_double(value_offset), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().mo_oracle_destroy(self.h)
            self.h = None

    def make_cache(self, x) -> Cache:
        x = _arr(x)
        h = C.c_void_p()
        _check(lib().mo_make_cache(self.h, _p(x), C.c_int64(x.size), C.byref(h)))
        return Cache(self, h)

    def value(self, cache: Cache) -> float:
        f = C.c_double()
        _check(lib().mo_value(self.h, cache.h, C.byref(f)))
        return f.value

    def moments(self, cache: Cache):
        out = np.empty(4)
        _check(lib().mo_moments(self.h, cache.h, _p(out)))
        return tuple(out)

    def gradient(self, cache: Cache) -> np.ndarray:
        g = np.empty(self.n)
        _check(lib().mo_gradient(self.h, cache.h, _p(g)))
        return g

    def hvp(self, cache: Cache, v) -> np.ndarray:
        v = _arr(v, self.n)
        out = np.empty(self.n)
        _check(lib().mo_hvp(self.h, cache.h, _p(v), _p(out)))
        return out

    def third_action(self, cache: Cache, u, v) -> np.ndarray:
        u, v = _arr(u, self.n), _arr(v, self.n)
        out = np.empty(self.n)
        _check(lib().mo_third_action(self.h, cache.h, _p(u), _p(v), _p(out)))
        return out

    def hessian_diag_weights(self, cache: Cache) -> np.ndarray:
        out = np.empty(self.T)
        _check(lib().mo_hessian_diag_weights(self.h, cache.h, _p(out)))
        return out

    def sample_direction(self, d) -> np.ndarray:
        d = _arr(d, self.n)
        out = np.empty(self.T)
        _check(lib().mo_sample_direction(self.h, _p(d), _p(out)))
        return out

    def line_model(self, cache: Cache, d, cap: float) -> np.ndarray:
        d = _arr(d)
        out = np.empty(14)
        _check(lib().mo_line_model(self.h, cache.h, _p(d), C.c_int64(d.size), C.c_double(cap), _p(out)))
        return out

    def passes(self):
        f, t = C.c_uint64(), C.c_uint64()
        lib().mo_passes(self.h, C.byref(f), C.byref(t))
        return f.value, t.value

    def reset_passes(self):
        lib().mo_reset_passes(self.h)

    def yand_direction(self, cache: Cache, cfg: mvsk_tangent_config, it_seed: int = 0):
        d = np.empty(self.n)
        diag = mvsk_direction_diag()
        _check(lib().mo_yand_direction(self.h, cache.h, C.byref(cfg), C.c_uint64(it_seed), _p(d), C.byref(diag)))
        return d, diag


def oracle_create_mu(A, mu):
    """Constructor with a mismatched mu length (oracle.hpp:37-38) -> raises."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    mu = _arr(mu)
    h = C.c_void_p()
    c = np.array([1.0, 1.0, 1.0, 1.0])
    _check(lib().mo_oracle_create_mu(_p(A), C.c_int64(A.shape[0]), C.c_int64(A.shape[1]), _p(mu),
                                     C.c_int64(mu.size), _p(c), C.byref(h)))
    lib().mo_oracle_destroy(h)


# ---- linesearch.hpp --------------------------------------------------------
def power_sums(z, w) -> np.ndarray:
    z, w = _arr(z), _arr(w)
    out = np.empty(9)
    _check(lib().mo_power_sums(_p(z), _p(w), C.c_int64(z.size), C.c_int64(w.size), _p(out)))
    return out


def cubic_real_roots(c3, c2, c1, c0) -> np.ndarray:
    out = np.empty(3)
    k = lib().mo_cubic_real_roots(*(C.c_double(v) for v in (c3, c2, c1, c0)), _p(out))
    return out[:k].copy()


def minimize_line(a, cap):
    a = _arr(a, 5)
    al, f = C.c_double(), C.c_double()
    _check(lib().mo_minimize_line(_p(a), C.c_double(cap), C.byref(al), C.byref(f)))
    return al.value, f.value


_PHI = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)


def armijo_search(phi, g_dot_d, alpha_init, sigma=1e-4, shrink=0.5):
    cb = _PHI(lambda a, _u: float(phi(a)))
    al, st = C.c_double(), C.c_int()
    _check(lib().mo_armijo(cb, None, C.c_double(g_dot_d), C.c_double(alpha_init), C.c_double(sigma),
                           C.c_double(shrink), C.byref(al), C.byref(st)))
    return al.value, bool(st.value)


# ---- simplex.hpp -----------------------------------------------------------
def alpha_max(x, d, tau) -> float:
    x, d = _arr(x), _arr(d)
    return lib().mo_alpha_max(_p(x), _p(d), x.size, tau)


def project_slice(v, tau, mass=1.0) -> np.ndarray:
    v = _arr(v)
    out = np.empty(v.size)
    _check(lib().mo_project_slice(_p(v), C.c_int64(v.size), C.c_double(tau), C.c_double(mass), _p(out)))
    return out


def projected_kkt_residual(g) -> float:
    g = _arr(g)
    return lib().mo_projected_kkt_residual(_p(g), g.size)


def gradient_mapping_residual(x, g, tau) -> float:
    x, g = _arr(x), _arr(g)
    return lib().mo_gradient_mapping_residual(_p(x), _p(g), x.size, tau)


def basis_apply(n, y) -> np.ndarray:
    y = _arr(y)
    out = np.empty(n)
    _check(lib().mo_basis_apply(C.c_int64(n), _p(y), C.c_int64(y.size), _p(out)))
    return out


def basis_apply_transpose(n, x) -> np.ndarray:
    x = _arr(x)
    out = np.empty(n - 1)
    _check(lib().mo_basis_apply_transpose(C.c_int64(n), _p(x), C.c_int64(x.size), _p(out)))
    return out


def householder_frame(g):
    g = _arr(g)
    m = g.size
    nu, v = np.empty(m), np.empty(m)
    beta, gn = C.c_double(), C.c_double()
    _check(lib().mo_householder_frame(_p(g), C.c_int64(m), _p(nu), _p(v), C.byref(beta), C.byref(gn)))
    return nu, v, beta.value, gn.value


def frame_apply_Q(g, eta) -> np.ndarray:
    g, eta = _arr(g), _arr(eta)
    out = np.empty(g.size)
    _check(lib().mo_frame_apply_Q(_p(g), C.c_int64(g.size), _p(eta), _p(out)))
    return out


def frame_apply_Qt(g, w) -> np.ndarray:
    g, w = _arr(g), _arr(w)
    out = np.empty(g.size - 1)
    _check(lib().mo_frame_apply_Qt(_p(g), C.c_int64(g.size), _p(w), _p(out)))
    return out


def cg_dense(M, rhs, tol, cap, jacobi=None):
    M = np.ascontiguousarray(M, dtype=np.float64)
    rhs = _arr(rhs)
    x = np.empty(rhs.size)
    it, bd = C.c_int(), C.c_int()
    jd = None if jacobi is None else _arr(jacobi)
    _check(lib().mo_cg_dense(_p(M), C.c_int64(rhs.size), _p(rhs), C.c_double(tol), C.c_int(cap), _p(jd),
                             _p(x), C.byref(it), C.byref(bd)))
    return x, it.value, bool(bd.value)


def restrict_to_face(A, mu, x, tau):
    A = np.ascontiguousarray(A, dtype=np.float64)
    T, n = A.shape
    mu, x = _arr(mu), _arr(x)
    idx = np.empty(n, dtype=np.int64)
    nf = C.c_int64()
    zoff = np.empty(T)
    mu_pin, free_mass = C.c_double(), C.c_double()
    _check(lib().mo_restrict_to_face(_p(A), C.c_int64(T), C.c_int64(n), _p(mu), _p(x), C.c_double(tau),
                                     idx.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(nf), _p(zoff),
                                     C.byref(mu_pin), C.byref(free_mass)))
    return idx[: nf.value].copy(), zoff, mu_pin.value, free_mass.value


# ---- solver.hpp ------------------------------------------------------------
def preset(name: str) -> mvsk_solver_config:
    cfg = mvsk_solver_config()
    _check(lib().mo_preset(name.encode(), C.byref(cfg)))
    return cfg


def solve(A, mu, coeffs, cfg: mvsk_solver_config, x0=None, observer=None):
    """solve(panel, coeffs, config, x0) (solver.hpp:195). Returns (x_star, report)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    T, n = A.shape
    mu, c = _arr(mu, n), _arr(coeffs, 4)
    xs = np.empty(n)
    rep = mvsk_solve_report()
    x0a = None if x0 is None else _arr(x0)
    if x0a is not None and x0a.size != n:
        # the reference validates the length inside solve (solver.hpp:220)
        raise OracleError(2, "solve: x0 is not in the tau-slice")
    if observer is not None:
        cb = OBSERVER_FN(lambda _u, it, f, xp, nn: observer(int(it), float(f), np.ctypeslib.as_array(xp, (nn,)).copy()))
    else:
        cb = OBSERVER_FN()
    _check(lib().mo_solve(_p(A), C.c_int64(T), C.c_int64(n), _p(mu), _p(c), C.byref(cfg), _p(x0a), _p(xs),
                          C.byref(rep), cb, None))
    return xs, rep


def tangent_config(mode="direct", lam=0.0, krylov_tol=1e-3, krylov_maxit=15, jacobi=False,
                   exact_trace=False, probes=8, probe_maxit=5) -> mvsk_tangent_config:
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
