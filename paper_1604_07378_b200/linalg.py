"""Prefactored SPD solves and the rotation-variant 3x3 SVD on the B200
(mirror of qnsim.linalg, linalg.py:1-110).

`Factorization` keeps the reference's duck type (`.n`, `.solve(B)`), so it can
replace `SimSystem.sysfact` in the unmodified reference loop; the factor is a
supernodal Cholesky (host C++, nested-dissection ordering) whose triangular
solves run on the device (`qn_factor_solve`).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse

from paper_1604_07378_b200 import _lib

SIGMA_CLAMP = 1e-10  # linalg.py:13
FACTORIZE_COUNT = 0  # linalg.py:16 — "factor once, solve many" instrumentation


class FactorizationError(Exception):
    """Matrix is not symmetric positive definite (linalg.py:20-21)."""


class Factorization:
    """Cholesky handle; immutable, unlimited solves (linalg.py:23-40)."""

    def __init__(self, A, coords=None, batch_values=None):
        _lib.require_gpu()
        if scipy.sparse.issparse(A):
            A = scipy.sparse.csr_matrix(A, dtype=np.float64)
        else:
            A = np.asarray(A, dtype=np.float64)
            if A.ndim != 2 or A.shape[0] != A.shape[1]:
                raise FactorizationError(f"expected square matrix, got shape {A.shape}")
            A = scipy.sparse.csr_matrix(A)
        if A.shape[0] != A.shape[1]:
            raise FactorizationError(f"expected square matrix, got shape {A.shape}")
        A.sort_indices()
        self.n = A.shape[0]
        indptr, indices = _lib.i64(A.indptr), _lib.i32(A.indices)
        vals = _lib.f64(A.data) if batch_values is None else _lib.f64(batch_values)
        nb = vals.size // max(A.nnz, 1) if batch_values is not None else 1
        xyz = None if coords is None else _lib.f64(coords)
        h = C.c_void_p()
        rc = _lib.load().qn_factor_create(self.n, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(vals), nb,
                                          _lib.ptr(xyz), C.byref(h))
        _lib.check(rc, "factorize")
        self._h = h
        self._owned = True
        self.nbatch = nb

    @classmethod
    def _borrow(cls, handle, n, nbatch):
        self = cls.__new__(cls)
        self._h, self.n, self.nbatch, self._owned = handle, n, nbatch, False
        return self

    @property
    def op_handle(self) -> int:
        """Integer handle for the torch custom ops (torch_ops.py)."""
        return int(self._h.value if hasattr(self._h, "value") else self._h)

    def info(self) -> dict:
        inf = _lib.FactorInfo()
        _lib.check(_lib.load().qn_factor_info_get(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in inf._fields_}

    def solve(self, B, batch: int = 0) -> np.ndarray:
        B = np.asarray(B, dtype=np.float64)
        if B.shape[0] != self.n:
            raise ValueError(f"rhs has {B.shape[0]} rows, factorization has dimension {self.n}")
        vec = B.ndim == 1
        B2 = _lib.f64(B.reshape(self.n, -1))
        X = np.empty_like(B2)
        _lib.check(_lib.load().qn_factor_solve(self._h, batch, _lib.ptr(B2), _lib.ptr(X), B2.shape[1],
                                               _lib.QN_MEM_HOST, None), "solve")
        return X.reshape(B.shape) if vec else X

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None):
            try:
                _lib.load().qn_factor_destroy(self._h)
            except Exception:
                pass
            self._h = None


def factorize_spd(A, coords=None) -> Factorization:
    """Factor once; the handle is reused for every solve (linalg.py:43-54)."""
    global FACTORIZE_COUNT
    fact = Factorization(A, coords=coords)
    FACTORIZE_COUNT += 1
    return fact


def solve_prefactored(F: Factorization, B: np.ndarray) -> np.ndarray:
    """linalg.py:57-59"""
    return F.solve(B)


@dataclass(frozen=True)
class RotVarSVD:
    """U, V proper rotations; reflection in sigma[2] (linalg.py:62-68)."""

    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray


def svd_rv_batch(F: np.ndarray):
    """Batched rotation-variant SVD on the GPU (linalg.py:86-110)."""
    F = _lib.f64(F)
    shape = F.shape[:-2]
    Fm = F.reshape(-1, 3, 3)
    m = Fm.shape[0]
    U = np.empty((m, 3, 3))
    V = np.empty((m, 3, 3))
    s = np.empty((m, 3))
    if m:
        _lib.require_gpu()
        _lib.check(_lib.load().qn_svd_rv_batch(m, _lib.ptr(Fm), _lib.ptr(U), _lib.ptr(s), _lib.ptr(V),
                                               _lib.QN_MEM_HOST, None), "svd")
    return U.reshape(shape + (3, 3)), s.reshape(shape + (3,)), V.reshape(shape + (3, 3))


def svd_rv(F: np.ndarray) -> RotVarSVD:
    """linalg.py:71-83"""
    F = np.asarray(F, dtype=np.float64)
    if F.shape != (3, 3):
        raise ValueError(f"expected 3x3 matrix, got {F.shape}")
    if not np.all(np.isfinite(F)):
        raise ValueError("non-finite entries in input matrix")
    U, s, V = svd_rv_batch(F[None])
    return RotVarSVD(U[0], s[0], V[0])
