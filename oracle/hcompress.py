"""Cluster tree, block tree, ACA and recompression (oracle restatement of
hmatrix.py:31-89, 179-264, 352-426)."""

from __future__ import annotations

import numpy as np


class Cluster:
    __slots__ = ("lo", "hi", "blo", "bhi", "kids", "level")

    def __init__(self, lo, hi, blo, bhi, level):
        self.lo, self.hi, self.blo, self.bhi, self.level = lo, hi, blo, bhi, level
        self.kids = []


def build_tree(points, C, n_leaf):
    """Median bisection on the longest bbox axis, stable sort (hmatrix.py:47-75).

    Returns (root, point permutation new->old, dof permutation new->old).
    """
    pts = np.asarray(points, float)
    perm = np.arange(pts.shape[0])

    def split(lo, hi, level):
        idx = perm[lo:hi]
        sub = pts[idx]
        node = Cluster(lo, hi, sub.min(0), sub.max(0), level)
        if (hi - lo) * C <= n_leaf or hi - lo < 2:
            return node
        ax = int(np.argmax(node.bhi - node.blo))
        perm[lo:hi] = idx[np.argsort(sub[:, ax], kind="stable")]
        mid = lo + (hi - lo) // 2
        node.kids = [split(lo, mid, level + 1), split(mid, hi, level + 1)]
        return node

    root = split(0, pts.shape[0], 0)
    dof_perm = (perm[:, None] * C + np.arange(C)).ravel()
    return root, perm, dof_perm


def box_diam(lo, hi):
    return float(np.linalg.norm(hi - lo))


def box_dist(a, b):
    gap = np.maximum(0.0, np.maximum(a.blo - b.bhi, b.blo - a.bhi))
    return float(np.linalg.norm(gap))


def is_admissible(a, b, eta):
    """dist > 0 and min diam <= eta dist (hmatrix.py:87-89)."""
    d = box_dist(a, b)
    return d > 0 and min(box_diam(a.blo, a.bhi), box_diam(b.blo, b.bhi)) <= eta * d


class Blk:
    """H-matrix node.  kind in {'H','D','R','LU'}; 'R' = low rank U@V."""
    __slots__ = ("kind", "r", "c", "kids", "D", "U", "V", "piv")

    def __init__(self, kind, r, c):
        self.kind, self.r, self.c = kind, r, c
        self.kids = None
        self.D = self.U = self.V = self.piv = None

    def rows(self):
        return self.r.kids or [self.r]

    def cols(self):
        return self.c.kids or [self.c]


def block_tree(root, eta):
    """Admissible -> 'R', leaf pairs -> 'D', else subdivide (hmatrix.py:194-204)."""
    def go(r, c):
        if is_admissible(r, c, eta):
            return Blk("R", r, c)
        if not r.kids and not c.kids:
            return Blk("D", r, c)
        b = Blk("H", r, c)
        b.kids = [[go(rk, ck) for ck in b.cols()] for rk in b.rows()]
        return b
    return go(root, root)


def leaves(b, out=None):
    out = [] if out is None else out
    if b.kind == "H":
        for row in b.kids:
            for k in row:
                leaves(k, out)
    else:
        out.append(b)
    return out


class Overflow(Exception):
    pass


def aca(get_row, get_col, m, n, tol, max_rank=None):
    """Partially pivoted ACA + recompression (hmatrix.py:352-409)."""
    budget = max(1, min(m, n) // 2) if max_rank is None else max_rank
    us, vs = [], []
    urow = np.zeros(m, bool)
    ucol = np.zeros(n, bool)
    f2 = 0.0
    i = 0
    while True:
        row = get_row(i)
        for u_l, v_l in zip(us, vs):
            row = row - u_l[i] * v_l
        urow[i] = True
        free = np.flatnonzero(~ucol)
        if free.size == 0:
            break
        j = int(free[np.argmax(np.abs(row[free]))])
        piv = row[j]
        if abs(piv) < 1e-300:
            rest = np.flatnonzero(~urow)
            if rest.size == 0:
                break
            i = int(rest[0])
            continue
        v = row / piv
        col = get_col(j)
        for u_l, v_l in zip(us, vs):
            col = col - v_l[j] * u_l
        ucol[j] = True
        u = col
        cross = sum(np.vdot(u_l, u) * (v @ np.conj(v_l)) for u_l, v_l in zip(us, vs))
        nu_, nv_ = np.linalg.norm(u), np.linalg.norm(v)
        f2 += 2.0 * float(np.real(cross)) + (nu_ * nv_) ** 2
        us.append(u)
        vs.append(v)
        if len(us) > budget:
            raise Overflow(len(us))
        if nu_ * nv_ <= tol * np.sqrt(max(f2, 0.0)):
            break
        rest = np.flatnonzero(~urow)
        if rest.size == 0:
            break
        i = int(rest[np.argmax(np.abs(u[rest]))])
    if not us:
        return np.zeros((m, 0), complex), np.zeros((0, n), complex)
    return truncate(np.stack(us, 1), np.stack(vs, 0), tol)


def truncate(U, V, tol):
    """QR(U), QR(V^T), SVD of the core, keep s > tol s0 (>=1) (hmatrix.py:412-426)."""
    if U.shape[1] == 0:
        return U, V
    Qu, Ru = np.linalg.qr(U)
    Qv, Rv = np.linalg.qr(V.T)
    W, s, Zh = np.linalg.svd(Ru @ Rv.T)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((U.shape[0], 0), U.dtype), np.zeros((0, V.shape[1]), V.dtype)
    r = max(1, int(np.sum(s > tol * s[0])))
    return Qu @ (W[:, :r] * s[:r]), Zh[:r] @ Qv.T


def svd_lowrank(P, tol):
    """Full SVD truncation of a dense update (hmatrix.py:605-609, 776-783)."""
    W, s, Zh = np.linalg.svd(P, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return None
    r = max(1, int(np.sum(s > tol * s[0])))
    return W[:, :r] * s[:r], Zh[:r]


class HMat:
    """Filled H-matrix: tree, permutation, root block (hmatrix.py:179-308)."""

    def __init__(self, points, C, n_leaf, eta):
        self.C = C
        self.root_cluster, self.pperm, self.dof_perm = build_tree(points, C, n_leaf)
        self.N = len(self.dof_perm)
        self.eta = eta
        self.root = block_tree(self.root_cluster, eta)
        self.demoted = 0

    def dofs(self, cl):
        return self.dof_perm[cl.lo * self.C: cl.hi * self.C]

    def fill(self, gen, tol, sample=None):
        """Dense leaves via gen.block, admissible via ACA (hmatrix.py:243-264).

        ``sample`` (optional index list) restricts work to those leaves, for
        bounded CPU-baseline timing.
        """
        lv = leaves(self.root)
        todo = range(len(lv)) if sample is None else sample
        for t in todo:
            b = lv[t]
            rows, cols = self.dofs(b.r), self.dofs(b.c)
            if b.kind == "D":
                b.D = gen.block(rows, cols)
                continue
            try:
                b.U, b.V = aca(lambda i: gen.row(int(rows[i]), cols),
                               lambda j: gen.col(rows, int(cols[j])),
                               rows.size, cols.size, tol)
            except Overflow:
                self.demoted += 1
                b.kind = "D"
                b.D = gen.block(rows, cols)
        return self

    def stored(self):
        tot = 0
        for b in leaves(self.root):
            tot += b.D.size if b.kind in ("D", "LU") else b.U.size + b.V.size
        return tot

    def compression_rate(self):
        return 1.0 - self.stored() / float(self.N) ** 2

    def to_dense(self):
        A = np.zeros((self.N, self.N), complex)
        C = self.C
        for b in leaves(self.root):
            M = b.D if b.kind == "D" else b.U @ b.V
            A[b.r.lo * C:b.r.hi * C, b.c.lo * C:b.c.hi * C] = M
        out = np.empty_like(A)
        out[np.ix_(self.dof_perm, self.dof_perm)] = A
        return out

    def matvec(self, x):
        xp = x[self.dof_perm]
        yp = np.zeros_like(xp)
        C = self.C
        for b in leaves(self.root):
            M = b.D if b.kind == "D" else None
            xs = xp[b.c.lo * C:b.c.hi * C]
            yp[b.r.lo * C:b.r.hi * C] += M @ xs if M is not None else b.U @ (b.V @ xs)
        y = np.empty_like(yp)
        y[self.dof_perm] = yp
        return y
