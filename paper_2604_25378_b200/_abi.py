"""ctypes mirror of include/mvsk_gpu.h (the C-ABI drop-in boundary).

Only the POD types and the loader live here. The library is built in-tree by
``__graft_entry__.build()`` into ``paper_2604_25378_b200/_build/libmvsk_b200.so``;
there is no CPU fallback — a missing library raises at load time.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
# MVSK_B200_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("MVSK_B200_LIB") or PKG_DIR / "_build" / "libmvsk_b200.so")

MVSK_GPU_ABI_VERSION = 1
MVSK_GPU_MAX_SLOTS = 8
MVSK_GPU_MAX_RHS = 16
MVSK_GPU_MAX_ASSETS = 8192
MVSK_NCCL_UNIQUE_ID_BYTES = 128

STATUS_NAMES = {
    0: "ok",
    1: "dimension_error",
    2: "domain_error",
    3: "data_error",
    4: "numeric_error",
    5: "cuda_error",
    6: "nccl_error",
    7: "internal_error",
}

SOLVE_STATUS = {0: "converged", 1: "stalled", 2: "max_iter", 3: "max_elapsed", 4: "degenerate_face"}


class mvsk_coeffs(C.Structure):
    _fields_ = [("c1", C.c_double), ("c2", C.c_double), ("c3", C.c_double), ("c4", C.c_double)]


class mvsk_tangent_config(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("krylov_maxit", C.c_int32),
        ("lambda_", C.c_double),
        ("krylov_tol", C.c_double),
        ("jacobi", C.c_int32),
        ("exact_trace", C.c_int32),
        ("hutchinson_probes", C.c_int32),
        ("probe_maxit", C.c_int32),
    ]


class mvsk_sweep_config(C.Structure):
    _fields_ = [("mean_tol", C.c_double), ("max_solves", C.c_int32), ("warm_start", C.c_int32)]


class mvsk_floor_point(C.Structure):
    _fields_ = [
        ("floor", C.c_double),
        ("c1", C.c_double),
        ("mean", C.c_double),
        ("f_star", C.c_double),
        ("kkt_residual", C.c_double),
        ("status", C.c_int32),
        ("solves", C.c_int32),
    ]


class mvsk_direction_diag(C.Structure):
    _fields_ = [
        ("reduced_grad_norm", C.c_double),
        ("u_norm", C.c_double),
        ("krylov_iters", C.c_int32),
        ("pcg_breakdown", C.c_int32),
        ("lambda_fallback", C.c_int32),
        ("_pad", C.c_int32),
    ]


class mvsk_solver_config(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("tau", C.c_double),
        ("max_iter", C.c_int32),
        ("has_max_elapsed", C.c_int32),
        ("max_elapsed_seconds", C.c_double),
        ("projected_trial_step", C.c_double),
        ("restart_trial_steps", C.c_double * 4),
        ("n_restart_trial_steps", C.c_int32),
        ("restart_max_iter", C.c_int32),
        ("tangent", mvsk_tangent_config),
        ("line_search", C.c_int32),
        ("stall_restarts", C.c_int32),
        ("identification_pass", C.c_int32),
        ("_pad", C.c_int32),
        ("label", C.c_char * 16),
    ]


class mvsk_solve_report(C.Structure):
    _fields_ = [
        ("f_star", C.c_double),
        ("kkt_residual", C.c_double),
        ("interior_residual", C.c_double),
        ("wall_seconds", C.c_double),
        ("krylov_iters_total", C.c_int64),
        ("oracle_passes", C.c_uint64),
        ("physical_passes", C.c_uint64),
        ("iterations", C.c_int32),
        ("face_events", C.c_int32),
        ("restarts", C.c_int32),
        ("identification_steps", C.c_int32),
        ("status", C.c_int32),
        ("_pad", C.c_int32),
        ("config_label", C.c_char * 16),
    ]


OBSERVER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_double, C.POINTER(C.c_double), C.c_int64)

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.c_int64
_I32 = C.c_int32
_U64P = C.POINTER(C.c_uint64)

# (name, restype, argtypes) for every symbol include/mvsk_gpu.h declares
SIGNATURES = [
    ("mvsk_gpu_abi_version", _I32, []),
    ("mvsk_gpu_status_string", C.c_char_p, [_I32]),
    ("mvsk_gpu_preset", _I32, [C.c_char_p, C.POINTER(mvsk_solver_config)]),
    ("mvsk_gpu_nccl_unique_id", _I32, [_P]),
    ("mvsk_gpu_create", _I32, [_D, _I64, _I64, _D, C.POINTER(mvsk_coeffs), _I32, C.POINTER(_P)]),
    ("mvsk_gpu_create_sharded", _I32,
     [_D, _I64, _I64, _I64, _I64, _D, C.POINTER(mvsk_coeffs), _I32, _I32, _I32, _P, C.POINTER(_P)]),
    ("mvsk_gpu_group_create", _I32, [_I32, C.POINTER(_P)]),
    ("mvsk_gpu_group_destroy", _I32, [_P]),
    ("mvsk_gpu_create_sharded_in_group", _I32,
     [_D, _I64, _I64, _I64, _I64, _D, C.POINTER(mvsk_coeffs), _I32, _P, _I32, C.POINTER(_P)]),
    ("mvsk_gpu_create_from_device", _I32,
     [_P, _I64, _I64, _I64, _I64, _I64, _D, C.POINTER(mvsk_coeffs), _I32, _I32, _I32, _P, C.POINTER(_P)]),
    ("mvsk_gpu_create_from_binary", _I32, [C.c_char_p, C.POINTER(mvsk_coeffs), _I32, _I32, _I32, _P, C.POINTER(_P)]),
    ("mvsk_gpu_binary_dims", _I32, [C.c_char_p, C.POINTER(_I64), C.POINTER(_I64)]),
    ("mvsk_gpu_mu", _I32, [_P, _D]),
    ("mvsk_gpu_destroy", _I32, [_P]),
    ("mvsk_gpu_last_error", C.c_char_p, [_P]),
    ("mvsk_gpu_set_stream", _I32, [_P, _P]),
    ("mvsk_gpu_synchronize", _I32, [_P]),
    ("mvsk_gpu_dims", _I32, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)]),
    ("mvsk_gpu_set_offset", _I32, [_P, _D, C.c_double]),
    ("mvsk_gpu_set_face", _I32, [_P, C.POINTER(_I64), _I64, C.c_double]),
    ("mvsk_gpu_make_cache", _I32, [_P, _I32, _D, _D]),
    ("mvsk_gpu_value", _I32, [_P, _I32, _D]),
    ("mvsk_gpu_moments", _I32, [_P, _I32, _D]),
    ("mvsk_gpu_gradient", _I32, [_P, _I32, _D]),
    ("mvsk_gpu_hvp", _I32, [_P, _I32, _D, _I32, _D]),
    ("mvsk_gpu_third_action", _I32, [_P, _I32, _D, _D, _I32, _D]),
    ("mvsk_gpu_hessian_diag_weights", _I32, [_P, _I32, _D]),
    ("mvsk_gpu_sample_direction", _I32, [_P, _D, _D]),
    ("mvsk_gpu_line_model", _I32, [_P, _I32, _D, C.c_double, _D]),
    ("mvsk_gpu_line_models", _I32, [_P, _I32, _D, _I32, _D]),
    ("mvsk_gpu_passes", _I32, [_P, _U64P, _U64P, _U64P]),
    ("mvsk_gpu_reset_passes", _I32, [_P]),
    ("mvsk_gpu_launch_count", _I32, [_P, _U64P]),
    ("mvsk_gpu_weighted_gram", _I32, [_P, _I32, _D]),
    ("mvsk_gpu_yand_direction", _I32,
     [_P, _I32, C.POINTER(mvsk_tangent_config), C.c_uint64, _D, C.POINTER(mvsk_direction_diag)]),
    ("mvsk_gpu_solve", _I32,
     [_P, C.POINTER(mvsk_solver_config), _D, _D, C.POINTER(mvsk_solve_report), OBSERVER_FN, _P]),
    ("mvsk_gpu_set_coeffs", _I32, [_P, C.POINTER(mvsk_coeffs)]),
    ("mvsk_gpu_floor_sweep", _I32,
     [_P, C.POINTER(mvsk_solver_config), C.POINTER(mvsk_sweep_config), _I32, _D, _D, C.POINTER(mvsk_floor_point),
      _D, _D, C.POINTER(_I32)]),
    ("mvsk_gpu_make_cache_device", _I32, [_P, _I32, _P]),
    ("mvsk_gpu_hvp_device", _I32, [_P, _I32, _P, _I32, _P]),
    ("mvsk_gpu_third_action_device", _I32, [_P, _I32, _P, _P, _I32, _P]),
    ("mvsk_gpu_line_sums_device", _I32, [_P, _I32, _P, _P]),
    ("mvsk_gpu_weighted_gram_device", _I32, [_P, _I32, _P]),
    ("mvsk_gpu_slot_pointers", _I32, [_P, _I32, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
]

_LIB = None


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load libmvsk_b200.so (built in-tree). Raises if it is missing: the
    product path has no CPU fallback."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libmvsk_b200.so not found at {p}; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA extension is required, there is no CPU fallback)")
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mvsk_gpu_abi_version() != MVSK_GPU_ABI_VERSION:
        raise RuntimeError("libmvsk_b200.so ABI version mismatch")
    if path is None:
        _LIB = lib
    return lib
