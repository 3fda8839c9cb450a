"""Patch geometry handed to the device (drop-in for chebscat.geometry's
Patch / CubeSphereFace / unit_sphere_patches, geometry.py:48-276).

Only host-side construction lives here: the node frames, Chebyshev
interpolants, charts and the closest-point Newton are evaluated on the GPU
(csrc/geometry.cuh, csrc/classify.cu).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

CHART_SAMPLES, CHART_CUBE_SPHERE, CHART_STAR = 0, 1, 2

_FACES = ((0, 1.0, 1, 2), (0, -1.0, 2, 1), (1, 1.0, 2, 0),
          (1, -1.0, 0, 2), (2, 1.0, 0, 1), (2, -1.0, 1, 0))


def fejer_nodes(n: int) -> np.ndarray:
    """First-kind Chebyshev points, descending (chebyshev.py:32-49)."""
    return np.cos((2.0 * np.arange(n) + 1.0) * np.pi / (2.0 * n))


@dataclass
class CubeSphereFace:
    """Cube face square projected on a sphere (geometry.py:48-97)."""
    radius: float
    face: int
    u_lo: float
    u_hi: float
    v_lo: float
    v_hi: float
    kind = CHART_CUBE_SPHERE

    def _cube(self, u, v):
        ax, sg, ua, va = _FACES[self.face]
        u = np.asarray(u, float)
        v = np.asarray(v, float)
        x = np.empty(np.broadcast(u, v).shape + (3,))
        x[..., ax] = sg
        x[..., ua] = self.u_lo + (u + 1.0) * 0.5 * (self.u_hi - self.u_lo)
        x[..., va] = self.v_lo + (v + 1.0) * 0.5 * (self.v_hi - self.v_lo)
        return x

    def positions(self, u, v):
        x = self._cube(u, v)
        return self.radius * x / np.linalg.norm(x, axis=-1, keepdims=True)

    def direction(self, u, v):
        x = self._cube(u, v)
        return x / np.linalg.norm(x, axis=-1, keepdims=True)

    def params(self) -> np.ndarray:
        return np.array([self.radius, self.face, self.u_lo, self.u_hi, self.v_lo, self.v_hi,
                         0.0, 0.0])


class _ShList:
    """Y[:, i] = value assignment sink for real_sh's polynomial mode."""

    def __init__(self, items):
        self.items = items

    def __setitem__(self, key, val):
        self.items[key[1]] = val


def real_sh(xyz, polys=None):
    """25 real orthonormal spherical harmonics l <= 4 at unit vectors (n,3);
    index l*l + (m+l).  With ``polys=(X, Y, Z)`` the same forms are built as
    _Poly objects (exact monomial expansion, star_tables)."""
    if polys is not None:
        x, y, z = polys
        Y = [None] * 25
    else:
        x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
        Y = np.empty((xyz.shape[0], 25))
    pi = np.pi
    Y0 = 0.5 * np.sqrt(1 / pi)
    if polys is not None:
        Y = _ShList(Y)
        Y[:, 0] = x * 0.0 + Y0
    else:
        Y[:, 0] = Y0
    c1 = np.sqrt(3 / (4 * pi))
    Y[:, 1], Y[:, 2], Y[:, 3] = c1 * y, c1 * z, c1 * x
    c2a, c2b, c2c = 0.5 * np.sqrt(15 / pi), 0.25 * np.sqrt(5 / pi), 0.25 * np.sqrt(15 / pi)
    Y[:, 4], Y[:, 5], Y[:, 6] = c2a * x * y, c2a * y * z, c2b * (3 * z * z - 1)
    Y[:, 7], Y[:, 8] = c2a * x * z, c2c * (x * x - y * y)
    c3a, c3b = 0.25 * np.sqrt(35 / (2 * pi)), 0.5 * np.sqrt(105 / pi)
    c3c, c3d, c3e = 0.25 * np.sqrt(21 / (2 * pi)), 0.25 * np.sqrt(7 / pi), 0.25 * np.sqrt(105 / pi)
    Y[:, 9] = c3a * y * (3 * x * x - y * y)
    Y[:, 10] = c3b * x * y * z
    Y[:, 11] = c3c * y * (5 * z * z - 1)
    Y[:, 12] = c3d * z * (5 * z * z - 3)
    Y[:, 13] = c3c * x * (5 * z * z - 1)
    Y[:, 14] = c3e * z * (x * x - y * y)
    Y[:, 15] = c3a * x * (x * x - 3 * y * y)
    c4a, c4b = 0.75 * np.sqrt(35 / pi), 0.75 * np.sqrt(35 / (2 * pi))
    c4c, c4d = 0.75 * np.sqrt(5 / pi), 0.75 * np.sqrt(5 / (2 * pi))
    c4e, c4f, c4g = (3 / 16) * np.sqrt(1 / pi), (3 / 8) * np.sqrt(5 / pi), (3 / 16) * np.sqrt(35 / pi)
    Y[:, 16] = c4a * x * y * (x * x - y * y)
    Y[:, 17] = c4b * y * z * (3 * x * x - y * y)
    Y[:, 18] = c4c * x * y * (7 * z * z - 1)
    Y[:, 19] = c4d * y * z * (7 * z * z - 3)
    Y[:, 20] = c4e * (35 * z ** 4 - 30 * z * z + 3)
    Y[:, 21] = c4d * x * z * (7 * z * z - 3)
    Y[:, 22] = c4f * (x * x - y * y) * (7 * z * z - 1)
    Y[:, 23] = c4b * x * z * (x * x - 3 * y * y)
    Y[:, 24] = c4g * (x * x * (x * x - 3 * y * y) - y * y * (3 * x * x - y * y))
    return Y.items if polys is not None else Y


def _monomials():
    """The 35 monomials x^a y^b z^c of degree <= 4, in the device's order."""
    return [(a, b, deg - a - b) for deg in range(5) for a in range(deg, -1, -1)
            for b in range(deg - a, -1, -1)]


class _Poly(dict):
    """Polynomial in x, y, z as {(a, b, c): coefficient} (exact expansion of real_sh)."""

    def __add__(self, o):
        o = o if isinstance(o, _Poly) else _Poly({(0, 0, 0): float(o)})
        r = _Poly(self)
        for k, v in o.items():
            r[k] = r.get(k, 0.0) + v
        return r

    __radd__ = __add__

    def __neg__(self):
        return _Poly({k: -v for k, v in self.items()})

    def __sub__(self, o):
        return self + (-o if isinstance(o, _Poly) else -float(o))

    def __rsub__(self, o):
        return (-self) + o

    def __mul__(self, o):
        if not isinstance(o, _Poly):
            return _Poly({k: v * o for k, v in self.items()})
        r = _Poly()
        for k1, v1 in self.items():
            for k2, v2 in o.items():
                k = (k1[0] + k2[0], k1[1] + k2[1], k1[2] + k2[2])
                r[k] = r.get(k, 0.0) + v1 * v2
        return r

    __rmul__ = __mul__

    def __pow__(self, n):
        r = _Poly({(0, 0, 0): 1.0})
        for _ in range(n):
            r = r * self
        return r

    def diff(self, axis):
        r = _Poly()
        for k, v in self.items():
            if k[axis]:
                kk = list(k)
                kk[axis] -= 1
                r[tuple(kk)] = r.get(tuple(kk), 0.0) + v * k[axis]
        return r


_STAR_TABLES: dict = {}


def star_tables(coef) -> np.ndarray:
    """[4 * 35] monomial coefficients of f = sum_i coef_i Y_i and of its Cartesian
    gradient (the CBIE_STAR_TABLE layout of include/cbie.h).  Y_i are real_sh's
    polynomial forms expanded exactly; the tables *define* the star chart on
    host and device alike."""
    key = np.asarray(coef, float).tobytes()
    if key in _STAR_TABLES:
        return _STAR_TABLES[key]
    X = _Poly({(1, 0, 0): 1.0})
    Y = _Poly({(0, 1, 0): 1.0})
    Z = _Poly({(0, 0, 1): 1.0})
    f = _Poly()
    for c, p in zip(np.asarray(coef, float), real_sh(None, polys=(X, Y, Z))):
        f = f + p * float(c)
    mons = _monomials()
    out = np.zeros((4, len(mons)))
    for t, poly in enumerate((f, f.diff(0), f.diff(1), f.diff(2))):
        for m, k in enumerate(mons):
            out[t, m] = poly.get(k, 0.0)
    _STAR_TABLES[key] = out.ravel()
    return _STAR_TABLES[key]


def _star_poly(F, px, py, pz):
    s = np.zeros_like(px[1])
    for m, (a, b, c) in enumerate(_monomials()):
        s = s + ((F[m] * px[a]) * py[b]) * pz[c]
    return s


def star_eval(a, face, ulo, uhi, vlo, vhi, tables, u, v):
    """Star chart position and tangents (csrc/geometry.cuh star_chart; every
    operation elementwise in the same order, so both round identically).
    u, v: 1-D arrays; returns (pos, a_u, a_v), each (n, 3)."""
    ax, sg, ua, va = _FACES[face]
    u = np.atleast_1d(np.asarray(u, float))
    v = np.atleast_1d(np.asarray(v, float))
    x = [None, None, None]
    x[ax] = np.full(u.shape, float(sg))
    x[ua] = ulo + ((u + 1.0) * 0.5) * (uhi - ulo)
    x[va] = vlo + ((v + 1.0) * 0.5) * (vhi - vlo)
    hu, hv = 0.5 * (uhi - ulo), 0.5 * (vhi - vlo)
    nrm = np.sqrt((x[0] * x[0] + x[1] * x[1]) + x[2] * x[2])
    xh = [xi / nrm for xi in x]
    tu = [((hu if i == ua else 0.0) - (xh[i] * xh[ua]) * hu) / nrm for i in range(3)]
    tv = [((hv if i == va else 0.0) - (xh[i] * xh[va]) * hv) / nrm for i in range(3)]
    one = np.ones(u.shape)
    px, py, pz = [one, xh[0]], [one, xh[1]], [one, xh[2]]
    for _ in range(3):
        px.append(px[-1] * xh[0])
        py.append(py[-1] * xh[1])
        pz.append(pz[-1] * xh[2])
    T = np.asarray(tables, float).reshape(4, 35)
    f = _star_poly(T[0], px, py, pz)
    gx = _star_poly(T[1], px, py, pz)
    gy = _star_poly(T[2], px, py, pz)
    gz = _star_poly(T[3], px, py, pz)
    r = a * (1.0 + f)
    dru = a * ((gx * tu[0] + gy * tu[1]) + gz * tu[2])
    drv = a * ((gx * tv[0] + gy * tv[1]) + gz * tv[2])
    pos = np.stack([r * xh[i] for i in range(3)], -1)
    au = np.stack([dru * xh[i] + r * tu[i] for i in range(3)], -1)
    av = np.stack([drv * xh[i] + r * tv[i] for i in range(3)], -1)
    return pos, au, av


@dataclass
class StarFace(CubeSphereFace):
    """Seeded smooth star-shaped body r(xhat) = a (1 + sum_i c_i Y_i(xhat)) xhat on a
    cube-sphere face (config 4; not expressible by the reference's API, built as
    a Chart per SURVEY.md section 7 hard part 6).  ``coef`` already carries the
    0.2 / max|sum c Y| normalisation; the chart is evaluated from its monomial
    tables (``star_tables``), identically on host and device."""
    coef: Optional[np.ndarray] = None
    kind = CHART_STAR

    def tables(self):
        t = getattr(self, "_tables", None)
        if t is None:
            t = self._tables = star_tables(self.coef)
        return t

    def positions(self, u, v):
        u = np.asarray(u, float)
        return star_eval(self.radius, self.face, self.u_lo, self.u_hi, self.v_lo, self.v_hi,
                         self.tables(), u.ravel(), np.asarray(v, float).ravel())[0].reshape(
                             u.shape + (3,))

    def derivatives(self, u, v):
        _, au, av = star_eval(self.radius, self.face, self.u_lo, self.u_hi, self.v_lo, self.v_hi,
                              self.tables(), u, v)
        return au, av


@dataclass
class Patch:
    """samples[l, k, :] at (u_l, v_k) plus optional chart (geometry.py:100-117)."""
    id: int
    samples: np.ndarray
    chart: object = None

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=float)
        if self.samples.ndim != 3 or self.samples.shape[2] != 3:
            raise ValueError("samples must be (N_u, N_v, 3)")

    @property
    def orders(self):
        return self.samples.shape[:2]

    @property
    def n_nodes(self):
        return self.samples.shape[0] * self.samples.shape[1]

    @property
    def diameter(self):
        p = self.samples.reshape(-1, 3)
        return float(np.linalg.norm(p.max(0) - p.min(0)))


def _charted(charts, order):
    nu, nv = order
    uu = np.tile(fejer_nodes(nu), nv)          # flat node k*nu + l
    vv = np.repeat(fejer_nodes(nv), nu)
    out = []
    for pid, ch in enumerate(charts):
        smp = ch.positions(uu, vv).reshape(nv, nu, 3).transpose(1, 0, 2).copy()
        out.append(Patch(pid, smp, chart=ch))
    return out


def sphere_patches(radius: float, edges, order) -> list[Patch]:
    """Cube-sphere patches over a face split ``edges`` (face-major, iu, iv)."""
    e = np.asarray(edges, float)
    charts = [CubeSphereFace(radius, f, e[iu], e[iu + 1], e[iv], e[iv + 1])
              for f in range(6) for iu in range(len(e) - 1) for iv in range(len(e) - 1)]
    return _charted(charts, order)


def unit_sphere_patches(radius: float, refinement: int, order) -> list[Patch]:
    """6 * 4^refinement projected-cube patches (geometry.py:252-276)."""
    if radius <= 0 or refinement < 0:
        raise ValueError("radius must be positive and refinement >= 0")
    return sphere_patches(radius, np.linspace(-1.0, 1.0, 2 ** refinement + 1), order)


def star_coefficients(seed: int, amplitude: float = 0.2, grid: int = 200) -> np.ndarray:
    """c_lm ~ N(0,1) from default_rng(seed), l = 0..4 (25 real coefficients),
    scaled so max |sum c Y| over a (grid x 2 grid) theta/phi grid is ``amplitude``."""
    rng = np.random.default_rng(seed)
    c = rng.standard_normal(25)
    th = np.linspace(0.0, np.pi, grid)
    ph = np.linspace(0.0, 2 * np.pi, 2 * grid, endpoint=False)
    T, Ph = np.meshgrid(th, ph, indexing="ij")
    xyz = np.stack([np.sin(T) * np.cos(Ph), np.sin(T) * np.sin(Ph), np.cos(T)], -1).reshape(-1, 3)
    dev = np.abs(real_sh(xyz) @ c).max()
    return c * (amplitude / dev), rng


def star_patches(a: float, refinement: int, order, coef) -> list[Patch]:
    e = np.linspace(-1.0, 1.0, 2 ** refinement + 1)
    charts = [StarFace(a, f, e[iu], e[iu + 1], e[iv], e[iv + 1], coef=np.asarray(coef))
              for f in range(6) for iu in range(len(e) - 1) for iv in range(len(e) - 1)]
    return _charted(charts, order)


def _vander(x, n):
    V = np.empty((x.size, n))
    V[:, 0] = 1.0
    if n > 1:
        V[:, 1] = x
    for k in range(2, n):
        V[:, k] = 2.0 * x * V[:, k - 1] - V[:, k - 2]
    return V


def _analysis(n):
    """(alpha_k / n) T_k(x_l), alpha_0 = 1 (chebyshev.py:94-98)."""
    alpha = np.full(n, 2.0)
    alpha[0] = 1.0
    return (alpha[:, None] / n) * _vander(fejer_nodes(n), n).T


def _dcoef(n):
    d = np.zeros((n, n))
    for k in range(1, n):
        for j in range(k - 1, -1, -2):
            d[j, k] = 2.0 * k
    d[0, :] *= 0.5
    return d


def cheb_coefficients(patches: list[Patch]) -> np.ndarray:
    """[P][6][3][nu][nv]: coefficients of position and its first/second
    parametric derivatives (chebyshev.py:133-140, 205-209, geometry.py:137-143,
    228-238), computed with numpy exactly as the reference does so interpolated
    positions on the device round identically."""
    nu, nv = patches[0].orders
    Au, Av = _analysis(nu), _analysis(nv)
    Du, Dv = _dcoef(nu), _dcoef(nv)
    out = np.empty((len(patches), 6, 3, nu, nv))
    for q, p in enumerate(patches):
        for i in range(3):
            c = Au @ p.samples[:, :, i] @ Av.T
            cu = Du @ c
            cv = c @ Dv.T
            out[q, :, i] = (c, cu, cv, Du @ cu, cu @ Dv.T, cv @ Dv.T)
    return out


def device_arrays(patches: list[Patch]):
    """(samples [P][nu][nv][3], chart kind [P], chart params [P][8], star coef) for the C-ABI."""
    orders = {p.orders for p in patches}
    if len(orders) != 1:
        raise ValueError("the device path needs uniform patch orders")
    smp = np.ascontiguousarray(np.stack([p.samples for p in patches]))
    kind = np.zeros(len(patches), np.int32)
    par = np.zeros((len(patches), 8))
    star = None
    for i, p in enumerate(patches):
        if p.chart is None:
            continue
        kind[i] = p.chart.kind
        par[i] = p.chart.params()
        if p.chart.kind == CHART_STAR:
            star = np.ascontiguousarray(p.chart.tables(), dtype=float)
    return smp, kind, par, star, np.ascontiguousarray(cheb_coefficients(patches))
