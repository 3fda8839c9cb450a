"""Patch geometry (oracle restatement of geometry.py).

A patch is (samples[l,k,3], chart or None).  Charted patches evaluate the
analytic chart for positions/first derivatives; the closest-point Newton
always takes second derivatives from the Chebyshev interpolant of the samples
(geometry.py:228-245).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import spectral as sp

# (fixed axis, sign, u axis, v axis) per cube face  (geometry.py:57-61)
FACES = ((0, 1.0, 1, 2), (0, -1.0, 2, 1), (1, 1.0, 2, 0),
         (1, -1.0, 0, 2), (2, 1.0, 0, 1), (2, -1.0, 1, 0))


@dataclass
class CubeFace:
    """Cube face square [u_lo,u_hi]x[v_lo,v_hi] projected on a sphere (geometry.py:48-97)."""
    radius: float
    face: int
    u_lo: float
    u_hi: float
    v_lo: float
    v_hi: float

    def _cube(self, u, v):
        ax, sg, ua, va = FACES[self.face]
        hu = 0.5 * (self.u_hi - self.u_lo)
        hv = 0.5 * (self.v_hi - self.v_lo)
        u = np.asarray(u, dtype=float)
        v = np.asarray(v, dtype=float)
        x = np.empty(np.broadcast(u, v).shape + (3,))
        x[..., ax] = sg
        x[..., ua] = self.u_lo + (u + 1.0) * hu
        x[..., va] = self.v_lo + (v + 1.0) * hv
        tu = np.zeros(3)
        tv = np.zeros(3)
        tu[ua] = hu
        tv[va] = hv
        return x, tu, tv

    def pos(self, u, v):
        x, _, _ = self._cube(u, v)
        return self.radius * x / np.linalg.norm(x, axis=-1, keepdims=True)

    def tangents(self, u, v):
        x, tu, tv = self._cube(u, v)
        nx = np.linalg.norm(x, axis=-1, keepdims=True)
        xh = x / nx
        s = self.radius / nx
        return (s * (tu - xh * (xh @ tu)[..., None]),
                s * (tv - xh * (xh @ tv)[..., None]))


@dataclass
class Surf:
    """One patch: samples[l,k,:] at (u_l, v_k) plus optional chart."""
    samples: np.ndarray
    chart: object = None
    _memo: dict = field(default_factory=dict, repr=False)

    @property
    def nu(self):
        return self.samples.shape[0]

    @property
    def nv(self):
        return self.samples.shape[1]

    @property
    def npts(self):
        return self.nu * self.nv

    def diameter(self):
        p = self.samples.reshape(-1, 3)
        return float(np.linalg.norm(p.max(0) - p.min(0)))

    def bbox(self):
        p = self.samples.reshape(-1, 3)
        return p.min(0), p.max(0)

    def coeffs(self):
        c = self._memo.get("c")
        if c is None:
            c = np.stack([sp.grid_to_coeffs(self.samples[:, :, i]) for i in range(3)], -1)
            self._memo["c"] = c
        return c

    def node_uv(self):
        xu, _ = sp.fejer(self.nu)
        xv, _ = sp.fejer(self.nv)
        return np.tile(xu, self.nv), np.repeat(xv, self.nu)      # flat k*nu+l

    def node_w(self):
        _, wu = sp.fejer(self.nu)
        _, wv = sp.fejer(self.nv)
        return (wv[:, None] * wu[None, :]).ravel()

    def frames(self, u, v):
        """(pos, a_u, a_v, sqrt_g) at parameter points (geometry.py:196-220)."""
        u = np.atleast_1d(np.asarray(u, dtype=float))
        v = np.atleast_1d(np.asarray(v, dtype=float))
        if self.chart is not None:
            pos = self.chart.pos(u, v)
            au, av = self.chart.tangents(u, v)
        else:
            c = self.coeffs()
            pos = np.stack([sp.clenshaw2d(c[:, :, i], u, v) for i in range(3)], 1)
            au = np.stack([sp.clenshaw2d(sp.diff_coeffs(c[:, :, i], 0), u, v) for i in range(3)], 1)
            av = np.stack([sp.clenshaw2d(sp.diff_coeffs(c[:, :, i], 1), u, v) for i in range(3)], 1)
        sg = np.linalg.norm(np.cross(au, av), axis=-1)
        if np.any(sg < 1e-14 * self.diameter() ** 2):
            raise ValueError("degenerate patch Jacobian")
        return pos, au, av, sg

    def node_frames(self):
        f = self._memo.get("nf")
        if f is None:
            f = self.frames(*self.node_uv())
            self._memo["nf"] = f
        return f

    def hessian_parts(self, u, v):
        """r_uu, r_uv, r_vv from the interpolant (geometry.py:228-245)."""
        t = self._memo.get("h")
        if t is None:
            c = self.coeffs()
            t = [[sp.diff_coeffs(sp.diff_coeffs(c[:, :, i], a), b) for i in range(3)]
                 for a, b in ((0, 0), (0, 1), (1, 1))]
            self._memo["h"] = t
        return tuple(np.stack([sp.clenshaw2d(ci, u, v) for ci in comp], 1) for comp in t)


def sphere_mesh(radius: float, nsub: int, order: tuple[int, int], edges=None):
    """Cube-sphere patches, face-major then iu then iv (geometry.py:252-276).

    ``edges`` overrides the uniform split (config 5 uses linspace(-1,1,21)).
    """
    nu, nv = order
    xu, _ = sp.fejer(nu)
    xv, _ = sp.fejer(nv)
    uu = np.tile(xu, nv)
    vv = np.repeat(xv, nu)
    e = np.linspace(-1.0, 1.0, nsub + 1) if edges is None else np.asarray(edges, float)
    out = []
    for f in range(6):
        for iu in range(len(e) - 1):
            for iv in range(len(e) - 1):
                ch = CubeFace(radius, f, e[iu], e[iu + 1], e[iv], e[iv + 1])
                smp = ch.pos(uu, vv).reshape(nv, nu, 3).transpose(1, 0, 2).copy()
                out.append(Surf(smp, ch))
    return out


class StarChart:
    """Config-4 star chart: the chart definition of paper_2408_17116_b200.geometry
    (star_tables / star_eval, pure numpy; the same chart the reference is run with in
    tests/golden/make_golden_big.py)."""

    def __init__(self, a, face, ulo, uhi, vlo, vhi, tables):
        self.box = (a, face, ulo, uhi, vlo, vhi)
        self.tables = tables

    def pos(self, u, v):
        from paper_2408_17116_b200.geometry import star_eval
        return star_eval(*self.box, self.tables, np.ravel(u), np.ravel(v))[0]

    def tangents(self, u, v):
        from paper_2408_17116_b200.geometry import star_eval
        _, au, av = star_eval(*self.box, self.tables, np.ravel(u), np.ravel(v))
        return au, av


def star_mesh(a: float, nsub: int, order: tuple[int, int], coef):
    from paper_2408_17116_b200.geometry import star_tables
    tab = star_tables(coef)
    nu, nv = order
    xu, _ = sp.fejer(nu)
    xv, _ = sp.fejer(nv)
    uu = np.tile(xu, nv)
    vv = np.repeat(xv, nu)
    e = np.linspace(-1.0, 1.0, nsub + 1)
    out = []
    for f in range(6):
        for iu in range(nsub):
            for iv in range(nsub):
                ch = StarChart(a, f, e[iu], e[iu + 1], e[iv], e[iv + 1], tab)
                smp = ch.pos(uu, vv).reshape(nv, nu, 3).transpose(1, 0, 2).copy()
                out.append(Surf(smp, ch))
    return out
