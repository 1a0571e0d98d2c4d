"""Device setup assembly for large tet meshes: the numpy
part of build_system — mesh.tet_diff_operators (mesh.py:200-216),
mesh.lumped_masses (mesh.py:178-197), the COO assembly of L
(dynamics.py:387-402) and A_free = (L + M/h^2)[free][:, free]
(dynamics.py:413) — computed by CUDA kernels (csrc/qn_setup.cu) and copied
back once.  build_system takes this path for single-instance meshes of at
least DEVICE_SETUP_MIN_TETS tets (configs[4]); smaller systems keep the numpy
assembly, whose L is bitwise the reference's (the device inverse is the
adjugate, so values agree to rounding)."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import scipy.sparse

from paper_1604_07378_b200 import _lib

DEVICE_SETUP_MIN_TETS = 1_000_000


def use_device(n_tets: int, n_inst: int) -> bool:
    forced = os.environ.get("QN_DEVICE_SETUP")
    if forced is not None:
        return forced == "1" and n_inst == 1
    return n_inst == 1 and n_tets >= DEVICE_SETUP_MIN_TETS


def assemble(verts, tets, density, k_of_tet, h, fixed, vol_eps):
    """G (m,4,3), vols (m), masses (n), L (scipy CSR n x n), A_free (CSR nf x nf)."""
    lib = _lib.load()
    _lib.require_gpu()
    verts = _lib.f64(verts)
    tets32 = _lib.i32(tets)
    kt = _lib.f64(k_of_tet)
    fixed32 = _lib.i32(np.asarray(fixed, dtype=np.int64))
    n, m = verts.shape[0], tets32.shape[0]
    h_ = C.c_void_p()
    _lib.check(lib.qn_setup_create(n, _lib.ptr(verts), m, _lib.ptr(tets32), float(density), _lib.ptr(kt), float(h),
                                   fixed32.size, _lib.ptr(fixed32), float(vol_eps), C.byref(h_)), "setup")
    try:
        nnz_l, nf, nnz_a = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(lib.qn_setup_sizes(h_, C.byref(nnz_l), C.byref(nf), C.byref(nnz_a)))
        G = np.empty((m, 4, 3))
        vols = np.empty(m)
        masses = np.empty(n)
        lp, li, lv = np.empty(n + 1, np.int64), np.empty(nnz_l.value, np.int32), np.empty(nnz_l.value)
        ap, ai, av = np.empty(nf.value + 1, np.int64), np.empty(nnz_a.value, np.int32), np.empty(nnz_a.value)
        _lib.check(lib.qn_setup_copy(h_, _lib.ptr(G), _lib.ptr(vols), _lib.ptr(masses), _lib.ptr(lp), _lib.ptr(li),
                                     _lib.ptr(lv), _lib.ptr(ap), _lib.ptr(ai), _lib.ptr(av)), "setup")
    finally:
        lib.qn_setup_destroy(h_)
    L = scipy.sparse.csr_matrix((lv, li, lp), shape=(n, n))
    A_free = scipy.sparse.csr_matrix((av, ai, ap), shape=(nf.value, nf.value))
    return G, vols, masses, L, A_free
