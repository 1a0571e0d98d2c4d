"""ctypes binding of libqnsim_b200.so (C-ABI declared in include/qnsim_b200.h).

There is no CPU fallback: importing a compute entry point without the built
library, or calling one without a CUDA device, raises `QnRuntimeError`.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QN_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("QN_LIB") or os.path.join(_HERE, "libqnsim_b200.so")

QN_OK = 0
QN_ERR_ARG = 1
QN_ERR_CUDA = 2
QN_ERR_NOT_SPD = 3
QN_ERR_ALLOC = 4
QN_ERR_ASCENT = 5
QN_ERR_UNSUPPORTED = 6

QN_MEM_HOST = 0
QN_MEM_DEVICE = 1

QN_FN_ZERO, QN_FN_POLY, QN_FN_LOG, QN_FN_HERMITE, QN_FN_SQDEV, QN_FN_ANISO = 0, 1, 2, 3, 4, 5
QN_MAX_COEF = 12
QN_MAX_KNOTS = 12
QN_MAX_M = 16


class QnRuntimeError(RuntimeError):
    """The CUDA library is missing, failed, or no GPU is present."""


class ScalarFn(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("n", C.c_int32),
        ("c", C.c_double * QN_MAX_COEF), ("dc", C.c_double * QN_MAX_COEF),
        ("xs", C.c_double * QN_MAX_KNOTS), ("ys", C.c_double * QN_MAX_KNOTS), ("ts", C.c_double * QN_MAX_KNOTS),
        ("alpha", C.c_double), ("beta", C.c_double), ("eps", C.c_double),
        ("f0", C.c_double), ("f1", C.c_double), ("f2", C.c_double),
    ]


class Material(C.Structure):
    _fields_ = [("a", ScalarFn), ("b", ScalarFn), ("c", ScalarFn), ("shift", C.c_double)]


class FactorInfo(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nnz_a", C.c_int64), ("nnz_l", C.c_int64), ("n_supernodes", C.c_int64),
        ("max_front", C.c_int64), ("tree_depth", C.c_int64), ("nbatch", C.c_int64),
        ("factor_seconds", C.c_double), ("flops", C.c_double), ("dense_top", C.c_int64),
        ("nnz_l_sparse", C.c_int64), ("sinv_stored", C.c_int64),
    ]


class SystemDesc(C.Structure):
    _fields_ = [
        ("n_verts", C.c_int64), ("n_tets", C.c_int64), ("n_inst", C.c_int64), ("n_mat", C.c_int64),
        ("tets", C.c_void_p), ("Dm_inv", C.c_void_p), ("vols", C.c_void_p), ("tet_mat", C.c_void_p),
        ("mats", C.c_void_p), ("masses", C.c_void_p),
        ("n_fixed", C.c_int64), ("fixed", C.c_void_p),
        ("h", C.c_double), ("gravity", C.c_double * 3), ("scale", C.c_double),
        ("a_nnz", C.c_int64), ("a_indptr", C.c_void_p), ("a_indices", C.c_void_p), ("a_values", C.c_void_p),
        ("free_coords", C.c_void_p),
        ("solver", C.c_int32), ("pcg_maxit", C.c_int32), ("pcg_tol", C.c_double),
        ("n_colliders", C.c_int64), ("colliders", C.c_void_p), ("w_col", C.c_double),
        ("element_kind", C.c_int32), ("pad_e", C.c_int32), ("dminv_stride", C.c_int64),
    ]


class Collider(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("p", C.c_double * 3), ("n", C.c_double * 3),
                ("r0", C.c_double), ("r1", C.c_double)]


QN_COL_HALFSPACE, QN_COL_SPHERE, QN_COL_TORUS = 0, 1, 2
QN_ELEM_TET, QN_ELEM_SPRING = 0, 1
QN_MAX_COLLIDERS = 4


class SlabDesc(C.Structure):
    _fields_ = [
        ("local", C.c_void_p), ("own_lo", C.c_int64), ("own_hi", C.c_int64), ("tet_own_lo", C.c_int64),
        ("pinned", C.c_void_p), ("a_nnz", C.c_int64), ("a_indptr", C.c_void_p), ("a_indices", C.c_void_p),
        ("a_values", C.c_void_p), ("n_ranks", C.c_int32), ("pcg_maxit", C.c_int32), ("pcg_tol", C.c_double),
    ]


class SolverConfigC(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("iterations", C.c_int32), ("m", C.c_int32), ("line_search", C.c_int32),
        ("gamma", C.c_double), ("alpha_init", C.c_double), ("alpha_shrink", C.c_double),
        ("rho", C.c_double), ("S", C.c_int32), ("lbfgs_init", C.c_int32),
    ]


class FrameRecord(C.Structure):
    _fields_ = [
        ("g0", C.c_void_p), ("g", C.c_void_p), ("ls_trials", C.c_void_p), ("alphas", C.c_void_p),
        ("cum_ms", C.c_void_p), ("status", C.c_void_p), ("fallbacks", C.c_void_p),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32

# name -> argtypes (restype is always int except qn_last_error)
SIGNATURES = {
    "qn_version": [],
    "qn_device_count": [_P],
    "qn_launch_count": [_P],
    "qn_svd_rv_batch": [_I64, _P, _P, _P, _P, _I32, _P],
    "qn_material_eval": [_P, _I64, _P, _P, _P, _I32, _P],
    "qn_factor_create": [_I64, _P, _P, _P, _I64, _P, _P],
    "qn_factor_info_get": [_P, _P],
    "qn_factor_solve": [_P, _I64, _P, _P, _I64, _I32, _P],
    "qn_factor_destroy": [_P],
    "qn_factor_task_counts": [_P, _P, _P],
    "qn_factor_trace_solve": [_P, _P, _P],
    "qn_system_create": [_P, _P],
    "qn_system_destroy": [_P],
    "qn_system_factor": [_P, _P],
    "qn_state_set": [_P, _P, _P, _I32, _P],
    "qn_state_get": [_P, _P, _P, _P, _I32, _P],
    "qn_frame_step": [_P, _P, _P, _P, _I32, _I32, _P],
    "qn_simulate_frame": [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _P],
    "qn_system_objective": [_P, _P, _P, _P, _P, _I32, _P],
    "qn_system_elements": [_P, _I64, _I64, _P, _P, _P, _I32, _P],
    "qn_system_set_graph_mode": [_P, _I32],
    "qn_system_set_precision": [_P, _I32],
    "qn_system_last_frame_ms": [_P, _P],
    "qn_system_last_frame_passes": [_P, _P],
    "qn_system_last_frame_cg_iterations": [_P, _P],
    "qn_system_amg_info": [_P, _P, C.c_int64],
    "qn_system_set_timeline": [_P, C.c_int32],
    "qn_system_set_fault": [_P, C.c_int32, C.c_int32],
    "qn_frame_records_device": [_P, C.c_int32, _P, _P, _P],
    "qn_setup_create": [C.c_int64, _P, C.c_int64, _P, C.c_double, _P, C.c_double, C.c_int64, _P, C.c_double, _P],
    "qn_setup_sizes": [_P, _P, _P, _P],
    "qn_setup_copy": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "qn_setup_destroy": [_P],
    "qn_system_timeline": [_P, _P, C.c_int64],
    "qn_system_solve_trace": [_P, _P, _P],
    "qn_system_time_kernel": [_P, _I32, _I32, _P, _P],
    "qn_newton_direction": [_P, _P, _P, C.c_double, C.c_double, _P, _I32, _P],
    "qn_newton_release": [_P],
    "qn_system_rest_hessian": [_P, _P, C.c_double, C.c_double],
    "qn_slab_create": [_P, _P],
    "qn_slab_destroy": [_P],
    "qn_slab_buffer": [_P, _I32, _P, _P],
    "qn_slab_stage": [_P, _I32, _P, _I32, _P],
    "qn_slab_pcg_status": [_P, _P, _P, _P],
    "qn_slab_set_coarse": [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P],
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise QnRuntimeError(
            f"{path} is missing: build it with `python -m paper_1604_07378_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    lib.qn_last_error.restype = C.c_char_p
    lib.qn_last_error.argtypes = []
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    _lib = lib
    return lib


def device_count() -> int:
    c = C.c_int32(0)
    load().qn_device_count(C.byref(c))
    return c.value


def launch_count() -> int:
    c = C.c_int64(0)
    load().qn_launch_count(C.byref(c))
    return c.value


def require_gpu():
    if device_count() < 1:
        raise QnRuntimeError("no CUDA device visible: the B200 path has no CPU fallback")


def check(rc: int, what: str = ""):
    """Map a QN_ERR_* code to the reference's exception types."""
    if rc == QN_OK:
        return
    msg = (load().qn_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == QN_ERR_NOT_SPD:
        from paper_1604_07378_b200.linalg import FactorizationError
        raise FactorizationError(text)
    if rc == QN_ERR_ASCENT:
        from paper_1604_07378_b200.solvers import SolverError
        raise SolverError(text)
    if rc == QN_ERR_ARG:
        raise ValueError(text)
    if rc == QN_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    raise QnRuntimeError(f"[{rc}] {text}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
