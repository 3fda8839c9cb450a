"""Recursive H-LU with formatted arithmetic (oracle restatement of
hmatrix.py:433-858).  Operates in place on an HMat copy."""

from __future__ import annotations

import copy

import numpy as np
import scipy.linalg as sla
from scipy.linalg import lapack

from .hcompress import Blk, svd_lowrank, truncate


class Singular(Exception):
    pass


def _span(parent_cl, kid_cl, C):
    return slice((kid_cl.lo - parent_cl.lo) * C, (kid_cl.hi - parent_cl.lo) * C)


def _shape(b, C):
    return (b.r.hi - b.r.lo) * C, (b.c.hi - b.c.lo) * C


def mul_right(b, X, C):
    """b @ X (hmatrix.py:433-451)."""
    if b.kind == "D":
        return b.D @ X
    if b.kind == "R":
        return b.U @ (b.V @ X)
    if b.kind == "LU":
        raise TypeError("factored block")
    out = np.zeros((_shape(b, C)[0], X.shape[1]), complex)
    for a, rk in enumerate(b.rows()):
        for k, ck in enumerate(b.cols()):
            out[_span(b.r, rk, C)] += mul_right(b.kids[a][k], X[_span(b.c, ck, C)], C)
    return out


def mul_left(X, b, C):
    """X @ b (hmatrix.py:454-472)."""
    if b.kind == "D":
        return X @ b.D
    if b.kind == "R":
        return (X @ b.U) @ b.V
    if b.kind == "LU":
        raise TypeError("factored block")
    out = np.zeros((X.shape[0], _shape(b, C)[1]), complex)
    for a, rk in enumerate(b.rows()):
        for k, ck in enumerate(b.cols()):
            out[:, _span(b.c, ck, C)] += mul_left(X[:, _span(b.r, rk, C)], b.kids[a][k], C)
    return out


def densify(b, C):
    """(hmatrix.py:475-499)."""
    if b.kind == "D":
        return b.D.copy()
    if b.kind == "R":
        return b.U @ b.V
    if b.kind == "LU":
        n = b.D.shape[0]
        A = (np.tril(b.D, -1) + np.eye(n)) @ np.triu(b.D)
        for k in range(n - 1, -1, -1):
            p = b.piv[k]
            if p != k:
                A[[k, p]] = A[[p, k]]
        return A
    out = np.zeros(_shape(b, C), complex)
    for a, rk in enumerate(b.rows()):
        for k, ck in enumerate(b.cols()):
            out[_span(b.r, rk, C), _span(b.c, ck, C)] = densify(b.kids[a][k], C)
    return out


def add_lr(t, U, V, C, tol):
    """t += U V, truncating at low-rank targets (hmatrix.py:535-554)."""
    if U.shape[1] == 0:
        return
    if t.kind == "D":
        t.D += U @ V
    elif t.kind == "R":
        t.U, t.V = truncate(np.concatenate([t.U, U], 1), np.concatenate([t.V, V], 0), tol)
    else:
        for a, rk in enumerate(t.rows()):
            for k, ck in enumerate(t.cols()):
                add_lr(t.kids[a][k], U[_span(t.r, rk, C)], V[:, _span(t.c, ck, C)], C, tol)


def add_full(t, P, C, tol):
    """t += P for a dense P (hmatrix.py:599-617)."""
    if t.kind == "D":
        t.D += P
    elif t.kind == "R":
        f = svd_lowrank(P, tol)
        if f is not None:
            add_lr(t, f[0], f[1], C, tol)
    else:
        for a, rk in enumerate(t.rows()):
            for k, ck in enumerate(t.cols()):
                add_full(t.kids[a][k], P[_span(t.r, rk, C), _span(t.c, ck, C)], C, tol)


def gemm_h(t, A, B, C, tol, sign=-1.0):
    """t += sign A B in formatted arithmetic (hmatrix.py:557-596)."""
    if A.kind == "R":
        if A.U.shape[1]:
            add_lr(t, sign * A.U, mul_left(A.V, B, C), C, tol)
        return
    if B.kind == "R":
        if B.U.shape[1]:
            add_lr(t, sign * mul_right(A, B.U, C), B.V, C, tol)
        return
    if A.kind == "D" and B.kind == "D":
        add_full(t, sign * (A.D @ B.D), C, tol)
    elif A.kind == "D":
        add_full(t, sign * mul_left(A.D, B, C), C, tol)
    elif B.kind == "D":
        add_full(t, sign * mul_right(A, B.D, C), C, tol)
    elif t.kind == "H":
        for a in range(len(t.rows())):
            for b in range(len(t.cols())):
                for k in range(len(A.cols())):
                    gemm_h(t.kids[a][b], A.kids[a][k], B.kids[k][b], C, tol, sign)
    else:
        U, V = _prod_lowrank(A, B, C, tol)
        add_lr(t, sign * U, V, C, tol)


def _prod_lowrank(A, B, C, tol):
    """Agglomerated low-rank form of A B for H x H into a leaf (hmatrix.py:620-642)."""
    m = (A.r.hi - A.r.lo) * C
    n = (B.c.hi - B.c.lo) * C
    Us, Vs = [], []
    for a, rk in enumerate(A.rows()):
        for b, ck in enumerate(B.cols()):
            tmp = Blk("R", rk, ck)
            tmp.U = np.zeros(((rk.hi - rk.lo) * C, 0), complex)
            tmp.V = np.zeros((0, (ck.hi - ck.lo) * C), complex)
            for k in range(len(A.cols())):
                gemm_h(tmp, A.kids[a][k], B.kids[k][b], C, tol, 1.0)
            r = tmp.U.shape[1]
            if r:
                Ub = np.zeros((m, r), complex)
                Ub[_span(A.r, rk, C)] = tmp.U
                Vb = np.zeros((r, n), complex)
                Vb[:, _span(B.c, ck, C)] = tmp.V
                Us.append(Ub)
                Vs.append(Vb)
    U = np.concatenate(Us, 1) if Us else np.zeros((m, 0), complex)
    V = np.concatenate(Vs, 0) if Vs else np.zeros((0, n), complex)
    return truncate(U, V, tol)


def _pivot(X, piv):
    X = X.copy()
    for k, p in enumerate(piv):
        if p != k:
            X[[k, p]] = X[[p, k]]
    return X


def lsolve(L, X, C):
    """X := L^{-1} X, unit lower with leaf pivots (hmatrix.py:658-674)."""
    if L.kind == "LU":
        return sla.solve_triangular(L.D, _pivot(X, L.piv), lower=True, unit_diagonal=True)
    out = X.copy()
    rs = L.rows()
    for k, rk in enumerate(rs):
        sk = _span(L.r, rk, C)
        out[sk] = lsolve(L.kids[k][k], out[sk], C)
        for i in range(k + 1, len(rs)):
            out[_span(L.r, rs[i], C)] -= mul_right(L.kids[i][k], out[sk], C)
    return out


def usolve(U, X, C):
    """X := U^{-1} X (hmatrix.py:677-692)."""
    if U.kind == "LU":
        return sla.solve_triangular(U.D, X, lower=False)
    out = X.copy()
    rs = U.rows()
    for k in range(len(rs) - 1, -1, -1):
        sk = _span(U.r, rs[k], C)
        for i in range(k + 1, len(rs)):
            out[sk] -= mul_right(U.kids[k][i], out[_span(U.r, rs[i], C)], C)
        out[sk] = usolve(U.kids[k][k], out[sk], C)
    return out


def rsolve(X, U, C):
    """X := X U^{-1} (hmatrix.py:695-710)."""
    if U.kind == "LU":
        return sla.solve_triangular(U.D, X.T, lower=False, trans="T").T
    out = X.copy()
    cs = U.cols()
    for k, ck in enumerate(cs):
        sk = _span(U.c, ck, C)
        for l in range(k):
            out[:, sk] -= mul_left(out[:, _span(U.c, cs[l], C)], U.kids[l][k], C)
        out[:, sk] = rsolve(out[:, sk], U.kids[k][k], C)
    return out


def _overwrite(b, X, C, tol):
    """(hmatrix.py:770-791)."""
    if b.kind == "D":
        b.D = X
    elif b.kind == "R":
        f = svd_lowrank(X, tol)
        if f is None:
            b.U = np.zeros((X.shape[0], 0), complex)
            b.V = np.zeros((0, X.shape[1]), complex)
        else:
            b.U, b.V = f
    else:
        for a, rk in enumerate(b.rows()):
            for k, ck in enumerate(b.cols()):
                _overwrite(b.kids[a][k], X[_span(b.r, rk, C), _span(b.c, ck, C)], C, tol)


def lsolve_blk(L, B, C, tol):
    """B := L^{-1} B (hmatrix.py:713-740)."""
    if B.kind == "R":
        B.U = lsolve(L, B.U, C)
    elif B.kind == "D":
        B.D = lsolve(L, B.D, C)
    elif L.kind == "LU":
        for b in range(len(B.cols())):
            lsolve_blk(L, B.kids[0][b], C, tol)
    elif len(B.rows()) == 1:
        _overwrite(B, lsolve(L, densify(B, C), C), C, tol)
    else:
        s = len(L.rows())
        for k in range(s):
            for b in range(len(B.cols())):
                lsolve_blk(L.kids[k][k], B.kids[k][b], C, tol)
            for i in range(k + 1, s):
                for b in range(len(B.cols())):
                    gemm_h(B.kids[i][b], L.kids[i][k], B.kids[k][b], C, tol)


def rsolve_blk(B, U, C, tol):
    """B := B U^{-1} (hmatrix.py:743-767)."""
    if B.kind == "R":
        B.V = rsolve(B.V, U, C)
    elif B.kind == "D":
        B.D = rsolve(B.D, U, C)
    elif U.kind == "LU":
        for a in range(len(B.rows())):
            rsolve_blk(B.kids[a][0], U, C, tol)
    elif len(B.cols()) == 1:
        _overwrite(B, rsolve(densify(B, C), U, C), C, tol)
    else:
        s = len(U.cols())
        for k in range(s):
            for l in range(k):
                for a in range(len(B.rows())):
                    gemm_h(B.kids[a][k], B.kids[a][l], U.kids[l][k], C, tol)
            for a in range(len(B.rows())):
                rsolve_blk(B.kids[a][k], U.kids[k][k], C, tol)


def _factor(b, C, tol):
    """(hmatrix.py:834-858)."""
    if b.kind == "D":
        lu, piv = sla.lu_factor(b.D, check_finite=False)
        rc, _ = lapack.zgecon(lu, np.linalg.norm(b.D, 1))
        if rc < 1e-14:
            raise Singular(rc)
        b.kind, b.D, b.piv = "LU", lu, piv
        return
    if b.kind != "H":
        raise TypeError("diagonal block must be dense or subdivided")
    s = len(b.rows())
    for k in range(s):
        _factor(b.kids[k][k], C, tol)
        for i in range(k + 1, s):
            rsolve_blk(b.kids[i][k], b.kids[k][k], C, tol)
        for j in range(k + 1, s):
            lsolve_blk(b.kids[k][k], b.kids[k][j], C, tol)
        for i in range(k + 1, s):
            for j in range(k + 1, s):
                gemm_h(b.kids[i][j], b.kids[i][k], b.kids[k][j], C, tol)


class Factors:
    def __init__(self, H, tol):
        self.H = H
        self.root = copy.deepcopy(H.root)
        _factor(self.root, H.C, tol)

    def solve(self, b):
        """(hmatrix.py:807-816)."""
        b = np.asarray(b, complex)
        one = b.ndim == 1
        B = b.reshape(-1, 1) if one else b
        X = usolve(self.root, lsolve(self.root, B[self.H.dof_perm], self.H.C), self.H.C)
        out = np.empty_like(X)
        out[self.H.dof_perm] = X
        return out[:, 0] if one else out
