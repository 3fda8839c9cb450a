"""Classification, graded singular rule, pair blocks, dense assembly.

Oracle restatement of quadrature.py (classify / closest_points /
build_singular_rule) and assembly.py (EntryGenerator pair blocks, block
access, assemble_dense, rhs).
"""

from __future__ import annotations

import numpy as np

from . import physics as ph
from . import spectral as sp

FAR, NEAR, SELF = 0, 1, 2
SCREEN_MARGIN = 1.25            # quadrature.py:28


def closest_points(surf, obs):
    """Damped lock-step Newton closest point (quadrature.py:87-140).

    Returns uv (m,2) clipped to [-1,1], distance (m,), converged flag (m,).
    """
    obs = np.atleast_2d(obs)
    m = obs.shape[0]
    nodes = surf.node_frames()[0]
    d2 = (np.einsum("mx,mx->m", obs, obs)[:, None] - 2.0 * obs @ nodes.T
          + np.einsum("nx,nx->n", nodes, nodes)[None, :])
    seed = np.argmin(d2, axis=1)
    un, vn = surf.node_uv()
    uv0 = np.stack([un[seed], vn[seed]], 1)
    uv = uv0.copy()
    live = np.ones(m, bool)
    ok = np.zeros(m, bool)
    for _ in range(30):
        idx = np.flatnonzero(live)
        if idx.size == 0:
            break
        pos, au, av, _sg = surf.frames(uv[idx, 0], uv[idx, 1])
        ruu, ruv, rvv = surf.hessian_parts(uv[idx, 0], uv[idx, 1])
        d = pos - obs[idx]
        dot = lambda a, b: np.einsum("mx,mx->m", a, b)   # noqa: E731
        g0, g1 = 2.0 * dot(au, d), 2.0 * dot(av, d)
        a00, a01, a11 = dot(au, au), dot(au, av), dot(av, av)
        h00 = 2.0 * (a00 + dot(ruu, d))
        h01 = 2.0 * (a01 + dot(ruv, d))
        h11 = 2.0 * (a11 + dot(rvv, d))
        det = h00 * h11 - h01 * h01
        gn = (det <= 1e-30) | (h00 <= 0)
        h00 = np.where(gn, 2.0 * a00, h00)
        h01 = np.where(gn, 2.0 * a01, h01)
        h11 = np.where(gn, 2.0 * a11, h11)
        det = np.where(gn, h00 * h11 - h01 * h01, det)
        su = -(h11 * g0 - h01 * g1) / det
        sv = -(-h01 * g0 + h00 * g1) / det
        new = np.clip(uv[idx] + np.stack([su, sv], 1), -1.05, 1.05)
        moved = np.abs(new - uv[idx]).max(axis=1)
        uv[idx] = new
        fin = moved < 1e-12
        ok[idx[fin]] = True
        live[idx[fin]] = False
    uv = np.where(ok[:, None], uv, uv0)
    uv = np.clip(uv, -1.0, 1.0)
    pos = surf.frames(uv[:, 0], uv[:, 1])[0]
    return uv, np.linalg.norm(pos - obs, axis=1), ok


def graded_rule(us, vs, n, p=3):
    """Corner-split graded tensor rule around (u*,v*) (quadrature.py:143-183)."""
    x, w = sp.fejer(n)
    sig = 0.5 * (x + 1.0)
    s = sig ** p
    ws = 0.5 * w * p * sig ** (p - 1)
    pts, wts = [], []
    for lo, hi in ((-1.0, us), (us, 1.0)):
        if abs(hi - lo) < 1e-12:
            continue
        fu = lo if lo != us else hi
        un, wu = us + s * (fu - us), ws * abs(fu - us)
        for vlo, vhi in ((-1.0, vs), (vs, 1.0)):
            if abs(vhi - vlo) < 1e-12:
                continue
            fv = vlo if vlo != vs else vhi
            vn, wv = vs + s * (fv - vs), ws * abs(fv - vs)
            pts.append(np.stack([np.repeat(un, n), np.tile(vn, n)], 1))
            wts.append(np.outer(wu, wv).ravel())
    return np.concatenate(pts), np.concatenate(wts)


class Discretisation:
    """Points, dof map, classification table and pair blocks for one problem.

    Restates assembly.py:41-61 (DofMap), 106-143 (classification), 146-226
    (pair blocks), 253-334 (block access) and 438-466 (dense, rhs).
    """

    def __init__(self, surfs, form: ph.Form, tau=1.0, oversample=None, grading=3):
        self.surfs = surfs
        self.form = form
        self.C = form.C
        self.tau = tau
        self.grading = grading
        counts = np.array([s.npts for s in surfs])
        self.off = np.concatenate([[0], np.cumsum(counts)])
        self.npts = int(self.off[-1])
        self.N = self.npts * self.C
        self.patch_of = np.repeat(np.arange(len(surfs)), counts)
        self.node_of = np.concatenate([np.arange(c) for c in counts])
        nf = [s.node_frames() for s in surfs]
        self.pos = np.concatenate([f[0] for f in nf])
        self.au = np.concatenate([f[1] for f in nf])
        self.av = np.concatenate([f[2] for f in nf])
        self.wg = [s.node_w() * f[3] for s, f in zip(surfs, nf)]
        self.nover = [oversample if oversample is not None else max(2 * max(s.nu, s.nv), 16)
                      for s in surfs]
        self.cls = {}           # (point, patch) -> (tag, u, v, ok) for non-FAR pairs
        self.done = set()
        self.fallbacks = 0
        self._memo = {}

    # -- classification (assembly.py:106-143) --------------------------------
    def classify_patch(self, q):
        if q in self.done:
            return
        s = self.surfs[q]
        lo, hi = s.bbox()
        diam = s.diameter()
        own = self.patch_of == q
        gap = np.maximum(0.0, np.maximum(lo - self.pos, self.pos - hi))
        screened = np.linalg.norm(gap, axis=1) >= self.tau * diam * SCREEN_MARGIN
        need = np.flatnonzero(~screened & ~own)
        if need.size:
            uv, dist, ok = closest_points(s, self.pos[need])
            self.fallbacks += int(np.sum(~ok))
            for a, p in enumerate(need):
                if dist[a] < self.tau * diam:
                    self.cls[(int(p), q)] = (NEAR, float(uv[a, 0]), float(uv[a, 1]), bool(ok[a]))
        un, vn = s.node_uv()
        for p in np.flatnonzero(own):
            n0 = int(self.node_of[p])
            self.cls[(int(p), q)] = (SELF, float(un[n0]), float(vn[n0]), True)
        self.done.add(q)

    def tag(self, p, q):
        self.classify_patch(q)
        return self.cls.get((p, q), (FAR, np.nan, np.nan, True))

    def classify_all(self):
        for q in range(len(self.surfs)):
            self.classify_patch(q)

    # -- pair blocks (assembly.py:170-226) -------------------------------------
    def pair_block(self, p, q):
        key = (p, q)
        hit = self._memo.get(key)
        if hit is not None:
            return hit
        out = self._pair(p, q)
        if len(self._memo) < 200000:
            self._memo[key] = out
        return out

    def _pair(self, p, q):
        f, C, s = self.form, self.C, self.surfs[q]
        nu, nv = s.nu, s.nv
        xo, auo, avo = self.pos[p], self.au[p], self.av[p]
        t, us, vs, _ = self.tag(p, q)
        if t == FAR:
            ys, aus, avs, sgs = s.node_frames()
            wg = self.wg[q]
            if C == 2:
                B = ph.mfie_block(f.outer.k, xo, auo, avo, ys, aus, avs, sgs)
                out = np.einsum("j,jbc->bjc", wg, B)
            else:
                Bv, Bd = ph.muller_expand(*ph.muller_fields(f, xo, auo, avo, ys, aus, avs, sgs))
                out = np.einsum("j,jbc->bjc", wg, Bv)
                out = out + self._div_far(q, (wg[:, None, None] * Bd).transpose(1, 0, 2))
        else:
            nodes, w = graded_rule(us, vs, self.nover[q], self.grading)
            ys, aus, avs, sgs = s.frames(nodes[:, 0], nodes[:, 1])
            keep = np.einsum("ij,ij->i", ys - xo, ys - xo) > 1e-28
            if not np.all(keep):
                ys, aus, avs, sgs = ys[keep], aus[keep], avs[keep], sgs[keep]
                nodes, w = nodes[keep], w[keep]
            P, Du, Dv = sp.cardinal(nu, nv, nodes[:, 0], nodes[:, 1])
            wg = w * sgs
            if C == 2:
                B = ph.mfie_block(f.outer.k, xo, auo, avo, ys, aus, avs, sgs)
                Y = (wg[:, None, None] * B).reshape(-1, 4)
                out = (Y.T @ P).reshape(2, 2, -1).transpose(0, 2, 1)
            else:
                T6, TdG = ph.muller_fields(f, xo, auo, avo, ys, aus, avs, sgs)
                W = ((T6 * wg[:, None, None]).reshape(-1, 12).T @ P).reshape(6, 2, -1)
                d = (TdG * wg[:, None]).T
                Wu, Wv = d @ Du, d @ Dv
                out = np.empty((4, nu * nv, 4), dtype=complex)
                out[0:2, :, 0] = W[0] + Wu
                out[0:2, :, 1] = W[1] + Wv
                out[0:2, :, 2] = W[2]
                out[0:2, :, 3] = W[3]
                out[2:4, :, 0] = W[4]
                out[2:4, :, 1] = W[5]
                out[2:4, :, 2] = W[0] + Wu
                out[2:4, :, 3] = W[1] + Wv
            out = np.array(out)
        if t == SELF:
            out[:, int(self.node_of[p]), :] += f.jump()
        return np.ascontiguousarray(out).reshape(C, nu * nv * C)

    def _div_far(self, q, Md):
        """Far-rule derivative columns through node diff matrices (assembly.py:215-226)."""
        s, C = self.surfs[q], self.C
        M4 = Md.reshape(C, s.nv, s.nu, C)
        o = np.zeros_like(M4)
        for c in range(C):
            if c % 2 == 0:
                o[..., c] = np.einsum("bkl,lm->bkm", M4[..., c], sp.node_diff(s.nu))
            else:
                o[..., c] = np.einsum("bkl,kn->bnl", M4[..., c], sp.node_diff(s.nv))
        return o.reshape(C, s.nv * s.nu, C)

    # -- access ------------------------------------------------------------------
    def entry(self, i, j):
        C = self.C
        p, b = divmod(int(i), C)
        pj, c = divmod(int(j), C)
        q = int(self.patch_of[pj])
        return self.pair_block(p, q)[b, int(self.node_of[pj]) * C + c]

    def block(self, rows, cols):
        """Sub-block through the canonical pair blocks (assembly.py:253-271)."""
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        C = self.C
        out = np.empty((rows.size, cols.size), dtype=complex)
        cp = cols // C
        cq = self.patch_of[cp]
        for q in np.unique(cq):
            sel = np.flatnonzero(cq == q)
            loc = self.node_of[cp[sel]] * C + cols[sel] % C
            for a, i in enumerate(rows):
                out[a, sel] = self.pair_block(int(i) // C, int(q))[int(i) % C, loc]
        return out

    def dense(self):
        """Full matrix (assembly.py:438-460)."""
        A = np.empty((self.N, self.N), dtype=complex)
        C = self.C
        for p in range(self.npts):
            for q in range(len(self.surfs)):
                blk = self.pair_block(p, q)
                lo = int(self.off[q]) * C
                A[p * C:(p + 1) * C, lo:lo + blk.shape[1]] = blk
        return A

    def rhs(self, direction, polarization, amplitude=1.0):
        """Tested plane-wave vector in dof order (assembly.py:463-466)."""
        r = ph.plane_wave_rows(self.form, direction, polarization, amplitude,
                               self.pos, self.au, self.av)
        return r.reshape(-1)

    def nclass(self):
        """(n_self, n_near) counts after classify_all."""
        tags = np.array([v[0] for v in self.cls.values()])
        return int(np.sum(tags == SELF)), int(np.sum(tags == NEAR))


class Scaled:
    """D_r A D_c generator over a Discretisation (solver.py:90-129)."""

    def __init__(self, disc: Discretisation):
        self.disc = disc
        rc, cc = disc.form.scales()
        self.row_scale = np.tile(rc, disc.npts)
        self.col_scale = np.tile(cc, disc.npts)

    def row(self, i, cols):
        cols = np.asarray(cols)
        return self.disc.block([i], cols)[0] * (self.row_scale[i] * self.col_scale[cols])

    def col(self, rows, j):
        rows = np.asarray(rows)
        return self.disc.block(rows, [j])[:, 0] * (self.row_scale[rows] * self.col_scale[j])

    def block(self, rows, cols):
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        return (self.disc.block(rows, cols) * self.row_scale[rows][:, None]
                * self.col_scale[cols][None, :])
