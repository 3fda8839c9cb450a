"""Device-resident H-matrix and H-LU factors (drop-in for chebscat.hmatrix's
HMatrix / hlu_factor / HLUFactors, hmatrix.py:179-308, 798-858).

The cluster tree, block tree, dense-leaf fill, batched ACA, recompression,
H-LU and solves all run in libcbie.so; these classes hold the handles.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _ffi


class HMatrix:
    """H-matrix of the equilibrated system D_r A D_c (solver.py:132-145)."""

    def __init__(self, gen, n_leaf: int, eta: float, aca_tol: float, shard=None):
        """shard = (rank, world, exchange): fill only this process's leaves (LPT
        partition); exchange=True broadcasts the shards over the context's NCCL
        communicator (dist.init_nccl) so every rank holds the complete H-matrix."""
        self.gen = gen                     # keeps the device context alive
        self.dev = gen.dev
        self.C = gen.C
        self.N = gen.n_dofs
        self.eta = eta
        self.aca_tol = aca_tol
        self.shard = shard
        h = ct.c_void_p()
        if shard is None:
            self.dev.check(self.dev.lib.cbie_hmatrix_build(self.dev.h, int(n_leaf), float(eta),
                                                           float(aca_tol), ct.byref(h)))
        else:
            rank, world, exchange = shard
            self.dev.check(self.dev.lib.cbie_hmatrix_build_shard(
                self.dev.h, int(n_leaf), float(eta), float(aca_tol), int(rank), int(world),
                int(bool(exchange)), ct.byref(h)))
        self.h = h
        self._stats = _ffi.stats(h, 1)

    @classmethod
    def from_generator(cls, points, C: int, n_leaf: int, eta: float, generator, tol: float,
                       device: int = 0) -> "HMatrix":
        """H-matrix of any host generator honouring the reference's protocol
        (``block(rows, cols)``, hmatrix.py:243-264), e.g. the reference test-suite's
        KernelGen / IdGen / ZeroGen (tests/test_hmatrix.py:9-36, 228-274): the cluster
        and block trees of ``points`` (build_cluster_tree / build_block_tree), every
        leaf's block evaluated through the generator on the host, dense leaves stored and
        admissible ones compressed on the device (truncated SVD at tol, demotion above
        the ACA budget; cbie_hmatrix_import)."""
        from .assembly import Device
        pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
        lib = _ffi.load()
        n = ct.c_int64()
        npts = pts.shape[0]
        _ffi.check(lib.cbie_hmatrix_layout(_ffi.ptr(pts), npts, int(C), int(n_leaf), float(eta), None, None,
                                           ct.byref(n)))
        perm = np.empty(npts * C, np.int64)
        lv = np.empty((n.value, 5), np.int64)
        _ffi.check(lib.cbie_hmatrix_layout(_ffi.ptr(pts), npts, int(C), int(n_leaf), float(eta), _ffi.ptr(perm),
                                           _ffi.ptr(lv), ct.byref(n)))
        blocks = [np.asarray(generator.block(perm[r0 * C:r1 * C], perm[c0 * C:c1 * C]), complex).ravel()
                  for r0, r1, c0, c1, _ in lv]
        data = np.ascontiguousarray(np.concatenate(blocks) if blocks else np.zeros(1, complex))
        self = cls.__new__(cls)
        self.gen = None
        self.dev = Device(device)
        self.C = int(C)
        self.N = npts * int(C)
        self.eta = eta
        self.aca_tol = tol
        self.shard = None
        h = ct.c_void_p()
        self.dev.check(lib.cbie_hmatrix_import(self.dev.h, _ffi.ptr(pts), npts, int(C), int(n_leaf), float(eta),
                                               float(tol), _ffi.ptr(data), ct.byref(h)))
        self.h = h
        self._stats = _ffi.stats(h, 1)
        return self

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.dev.lib.cbie_hmatrix_destroy(h)
            self.h = None

    def offload(self) -> None:
        """Move the leaf data to pinned host memory mapped into the device address space
        (cbie_hmatrix_offload): the H-LU and matvec still read it, over the host link, and
        the device memory is free for the factorisation of problems too large for both
        (config 5: 67 GB H-matrix + the factors)."""
        self.dev.check(self.dev.lib.cbie_hmatrix_offload(self.h))

    # -- structure -------------------------------------------------------------------
    def tree(self):
        n = ct.c_int64()
        self.dev.check(self.dev.lib.cbie_hmatrix_tree(self.h, None, None, ct.byref(n)))
        perm = np.empty(self.N, np.int64)
        lv = np.empty((n.value, 6), np.int64)
        self.dev.check(self.dev.lib.cbie_hmatrix_tree(self.h, _ffi.ptr(perm), _ffi.ptr(lv),
                                                      ct.byref(n)))
        return perm, lv

    @property
    def dof_perm(self):
        return self.tree()[0]

    def leaf(self, i: int):
        """('dense', D) or ('lowrank', U, V) in permuted local order; ('remote',) for a
        leaf another shard filled (partial H-matrix before the exchange)."""
        perm, lv = self.tree()
        m = int(lv[i, 1] - lv[i, 0]) * self.C
        n = int(lv[i, 3] - lv[i, 2]) * self.C
        kind, rank = ct.c_int(), ct.c_int()
        self.dev.check(self.dev.lib.cbie_hmatrix_leaf(self.h, int(i), ct.byref(kind),
                                                      ct.byref(rank), None, None))
        if kind.value < 0:
            return ("remote",)
        if kind.value == 0:
            D = np.empty((m, n), complex)
            self.dev.check(self.dev.lib.cbie_hmatrix_leaf(self.h, int(i), ct.byref(kind),
                                                          ct.byref(rank), _ffi.ptr(D), None))
            return ("dense", D)
        r = rank.value
        U = np.empty((m, r), complex)
        V = np.empty((r, n), complex)
        self.dev.check(self.dev.lib.cbie_hmatrix_leaf(self.h, int(i), ct.byref(kind),
                                                      ct.byref(rank), _ffi.ptr(U), _ffi.ptr(V)))
        return ("lowrank", U, V)

    def to_dense(self) -> np.ndarray:
        """Dense reconstruction in ORIGINAL dof order (tests / diagnostics)."""
        perm, lv = self.tree()
        C = self.C
        A = np.zeros((self.N, self.N), complex)
        for i, row in enumerate(lv):
            lf = self.leaf(i)
            M = lf[1] if lf[0] == "dense" else lf[1] @ lf[2]
            A[row[0] * C:row[1] * C, row[2] * C:row[3] * C] = M
        out = np.empty_like(A)
        out[np.ix_(perm, perm)] = A
        return out

    # -- application / accounting ----------------------------------------------------------
    def matvec(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, complex)
        one = x.ndim == 1
        X = np.ascontiguousarray(x.reshape(-1, 1) if one else x)
        Y = np.empty_like(X)
        self.dev.check(self.dev.lib.cbie_hmatvec(self.h, _ffi.ptr(X), _ffi.ptr(Y), X.shape[1]))
        return Y[:, 0] if one else Y

    def stats(self) -> dict:
        return dict(self._stats)

    @property
    def demoted(self) -> int:
        return int(self._stats.get("demoted", 0))

    def stored_scalars(self) -> int:
        return int(self._stats["stored_scalars"])

    def memory_bytes(self) -> int:
        return self.stored_scalars() * 16

    def compression_rate(self) -> float:
        return 1.0 - self.stored_scalars() / float(self.N) ** 2

    def diagnostics(self) -> dict:
        """Per-level leaf counts, rank histogram, memory by leaf kind (HMatrix.diagnostics,
        hmatrix.py:290-308; same keys)."""
        perm, lv = self.tree()
        npts = self.N // self.C
        ranks: dict[int, int] = {}
        levels: dict[int, dict[str, int]] = {}
        mem = {"dense": 0, "lowrank": 0}
        for row in lv:
            lo, hi, lvl = 0, npts, 0          # depth of the row cluster (median split, hmatrix.py:62-75)
            while (lo, hi) != (int(row[0]), int(row[1])):
                mid = lo + (hi - lo) // 2
                lo, hi = (lo, mid) if row[0] < mid else (mid, hi)
                lvl += 1
            m, n = int(row[1] - row[0]) * self.C, int(row[3] - row[2]) * self.C
            kind = "lowrank" if row[4] == 1 else "dense"
            lk = levels.setdefault(lvl, {})
            lk[kind] = lk.get(kind, 0) + 1
            if row[4] == 1:
                r = int(row[5])
                ranks[r] = ranks.get(r, 0) + 1
                mem["lowrank"] += (m + n) * r * 16
            else:
                mem["dense"] += m * n * 16
        return {"levels": {str(k): v for k, v in sorted(levels.items())},
                "rank_histogram": {str(k): v for k, v in sorted(ranks.items())},
                "memory_bytes": mem,
                "compression_rate": self.compression_rate(),
                "demoted_blocks": self.demoted,
                "n_leaves": int(lv.shape[0])}


class HLUFactors:
    """H-LU factors on the device (HLUFactors, hmatrix.py:798-824)."""

    def __init__(self, H: HMatrix, tol: float, *, distributed: bool = False, emulate_world: int = 0):
        """distributed: block-row-distributed H-LU over the context's NCCL
        communicator (dist.init_nccl first; collective over the ranks);
        emulate_world > 0: the same distributed plan run by that many virtual
        ranks on this GPU (plan check without several GPUs)."""
        self.H = H
        self.dev = H.dev
        h = ct.c_void_p()
        lib = self.dev.lib
        if emulate_world:
            self.dev.check(lib.cbie_hlu_factor_emulated(H.h, float(tol), int(emulate_world), ct.byref(h)))
        elif distributed:
            self.dev.check(lib.cbie_hlu_factor_dist(H.h, float(tol), ct.byref(h)))
        else:
            self.dev.check(lib.cbie_hlu_factor(H.h, float(tol), ct.byref(h)))
        self.h = h
        self._stats = _ffi.stats(h, 2)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.dev.lib.cbie_hlu_destroy(h)
            self.h = None

    def solve(self, b: np.ndarray) -> np.ndarray:
        b = np.asarray(b, complex)
        one = b.ndim == 1
        B = np.ascontiguousarray(b.reshape(-1, 1) if one else b)
        X = np.empty_like(B)
        self.dev.check(self.dev.lib.cbie_hlu_solve(self.h, _ffi.ptr(B), _ffi.ptr(X), B.shape[1]))
        return X[:, 0] if one else X

    def stats(self) -> dict:
        return dict(self._stats)

    def stored_scalars(self) -> int:
        """Scalars held by the factors (HLUFactors.stored_scalars, hmatrix.py:818-821)."""
        return int(self._stats["stored_scalars"])

    def memory_bytes(self) -> int:
        return self.stored_scalars() * 16

    def solve_stats(self) -> dict:
        """Device statistics of the last solve (levels, launches, device ms)."""
        return {k: v for k, v in _ffi.stats(self.h, 2).items() if k.startswith("solve_")}

    def leaf(self, i: int):
        """('dense', D) | ('lu', LU, piv) | ('lowrank', U, V) for leaf i (permuted order)."""
        perm, lv = self.H.tree()
        C = self.H.C
        m = int(lv[i, 1] - lv[i, 0]) * C
        n = int(lv[i, 3] - lv[i, 2]) * C
        kind, rank = ct.c_int(), ct.c_int()
        self.dev.check(self.dev.lib.cbie_hlu_leaf(self.h, int(i), ct.byref(kind), ct.byref(rank),
                                                  None, None, None))
        if kind.value in (0, 2):
            D = np.empty((m, n), complex)
            piv = np.empty(m, np.int32)
            self.dev.check(self.dev.lib.cbie_hlu_leaf(self.h, int(i), ct.byref(kind), ct.byref(rank),
                                                      _ffi.ptr(D), None, _ffi.ptr(piv)))
            return ("lu", D, piv) if kind.value == 2 else ("dense", D)
        r = rank.value
        U = np.empty((m, r), complex)
        V = np.empty((r, n), complex)
        self.dev.check(self.dev.lib.cbie_hlu_leaf(self.h, int(i), ct.byref(kind), ct.byref(rank),
                                                  _ffi.ptr(U), _ffi.ptr(V), None))
        return ("lowrank", U, V)


def hlu_factor(H: HMatrix, tol: float, **kw) -> HLUFactors:
    return HLUFactors(H, tol, **kw)
