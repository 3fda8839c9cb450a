"""truncate_lowrank on the GPU (drop-in for hmatrix.truncate_lowrank,
hmatrix.py:412-426, and the dense SVD truncation of hmatrix.py:605-609)."""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _ffi
from .assembly import Device

_dev = None


def _device():
    global _dev
    if _dev is None:
        _dev = Device(0)
    return _dev


def truncate_lowrank(U: np.ndarray, V: np.ndarray, tol: float):
    """(U, V) -> recompressed (U', V') keeping s > tol s_0 (>= 1)."""
    d = _device()
    U = np.ascontiguousarray(U, complex)
    V = np.ascontiguousarray(V, complex)
    m, k = U.shape
    n = V.shape[1]
    if k == 0:
        return U, V
    cap = min(m, n, k)
    Uo = np.empty((m, cap), complex)
    Vo = np.empty((cap, n), complex)
    r = ct.c_int()
    d.check(d.lib.cbie_lowrank_truncate(d.h, _ffi.ptr(U), m, k, _ffi.ptr(V), n, float(tol),
                                        ct.byref(r), _ffi.ptr(Uo), _ffi.ptr(Vo)))
    rr = r.value
    return (np.ascontiguousarray(Uo.reshape(-1)[:m * rr].reshape(m, rr)),
            np.ascontiguousarray(Vo.reshape(-1)[:rr * n].reshape(rr, n)))


def svd_truncate(P: np.ndarray, tol: float):
    """Dense P -> (W_r s_r, Z_r^H) with s > tol s_0, or None if P == 0."""
    d = _device()
    P = np.ascontiguousarray(P, complex)
    m, n = P.shape
    cap = min(m, n)
    Uo = np.empty((m, cap), complex)
    Vo = np.empty((cap, n), complex)
    r = ct.c_int()
    d.check(d.lib.cbie_lowrank_truncate(d.h, _ffi.ptr(P), m, n, None, n, float(tol),
                                        ct.byref(r), _ffi.ptr(Uo), _ffi.ptr(Vo)))
    rr = r.value
    if rr == 0:
        return None
    return (np.ascontiguousarray(Uo.reshape(-1)[:m * rr].reshape(m, rr)),
            np.ascontiguousarray(Vo.reshape(-1)[:rr * n].reshape(rr, n)))
