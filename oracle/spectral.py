"""Chebyshev / Fejer-1 tables (oracle restatement of chebyshev.py).

Grids are first-kind Chebyshev points x_l = cos((2l+1)pi/(2n)), i.e. in
DESCENDING order.  Everything is float64.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np


@lru_cache(maxsize=None)
def fejer(n: int):
    """Fejer-1 nodes and weights on [-1,1]  (chebyshev.py:32-49)."""
    if n < 1:
        raise ValueError("order must be >= 1")
    theta = (2.0 * np.arange(n) + 1.0) * np.pi / (2.0 * n)
    acc = np.ones(n)
    for m in range(1, n // 2 + 1):
        acc -= 2.0 * np.cos(2 * m * theta) / (4 * m * m - 1)
    return np.cos(theta), (2.0 / n) * acc


def vander(x, n: int) -> np.ndarray:
    """T_k(x_i), k < n, by the three-term recurrence (chebyshev.py:52-61)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    out = np.empty((x.size, n))
    out[:, 0] = 1.0
    if n > 1:
        out[:, 1] = x
    for k in range(2, n):
        out[:, k] = 2.0 * x * out[:, k - 1] - out[:, k - 2]
    return out


def dvander(x, n: int) -> np.ndarray:
    """T_k'(x_i) = k U_{k-1}(x_i) (chebyshev.py:64-79)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    out = np.zeros((x.size, n))
    if n > 1:
        u_km2 = np.ones_like(x)
        out[:, 1] = u_km2
        u_km1 = 2.0 * x
        for k in range(2, n):
            out[:, k] = k * u_km1
            u_km2, u_km1 = u_km1, 2.0 * x * u_km1 - u_km2
    return out


@lru_cache(maxsize=None)
def analysis(n: int) -> np.ndarray:
    """Values -> coefficients, (alpha_k/n) T_k(x_l), alpha_0=1 else 2 (chebyshev.py:94-98)."""
    x, _ = fejer(n)
    alpha = np.full(n, 2.0)
    alpha[0] = 1.0
    return (alpha[:, None] / n) * vander(x, n).T


@lru_cache(maxsize=None)
def coef_diff(n: int) -> np.ndarray:
    """Coefficient-space d/dx (chebyshev.py:99-104)."""
    d = np.zeros((n, n))
    for k in range(1, n):
        d[k - 1::-2, k] = 2.0 * k
    d[0, :] *= 0.5
    return d


@lru_cache(maxsize=None)
def node_diff(n: int) -> np.ndarray:
    """Node-to-node spectral differentiation (chebyshev.py:105, 212-214)."""
    x, _ = fejer(n)
    return vander(x, n) @ coef_diff(n) @ analysis(n)


def grid_to_coeffs(vals: np.ndarray) -> np.ndarray:
    """gamma[n,m] of a [l,k] value grid (chebyshev.py:133-140)."""
    nu, nv = vals.shape
    return analysis(nu) @ vals @ analysis(nv).T


def diff_coeffs(c: np.ndarray, axis: int) -> np.ndarray:
    """d/du (axis 0) or d/dv (axis 1) of a coefficient tensor (chebyshev.py:205-209)."""
    if axis == 0:
        return coef_diff(c.shape[0]) @ c
    return c @ coef_diff(c.shape[1]).T


def clenshaw2d(c: np.ndarray, u, v) -> np.ndarray:
    """sum c[n,m] T_n(u) T_m(v) by Clenshaw, v first then u (chebyshev.py:163-202).

    The recurrence order is kept because the closest-point Newton (whose
    convergence flag decides the near rule) consumes these values.
    """
    u = np.atleast_1d(np.asarray(u, dtype=float))
    v = np.atleast_1d(np.asarray(v, dtype=float))
    ct = c.T                                    # (N_v, N_u)
    nv = ct.shape[0]
    vv = v[:, None]
    b1 = np.zeros((v.size, ct.shape[1]))
    b2 = np.zeros_like(b1)
    for k in range(nv - 1, 0, -1):
        b1, b2 = ct[k] + 2.0 * vv * b1 - b2, b1
    inner = ct[0] + vv * b1 - b2                # (npts, N_u)
    nu = inner.shape[1]
    b1 = np.zeros(u.size)
    b2 = np.zeros(u.size)
    for k in range(nu - 1, 0, -1):
        b1, b2 = inner[:, k] + 2.0 * u * b1 - b2, b1
    return inner[:, 0] + u * b1 - b2


def cardinal(nu: int, nv: int, u, v):
    """P, dP/du, dP/dv at points; column k*nu+l is node (l,k) (chebyshev.py:217-236)."""
    pu = vander(u, nu) @ analysis(nu)
    pv = vander(v, nv) @ analysis(nv)
    dpu = dvander(u, nu) @ analysis(nu)
    dpv = dvander(v, nv) @ analysis(nv)
    npts = pu.shape[0]
    P = (pv[:, :, None] * pu[:, None, :]).reshape(npts, -1)
    Du = (pv[:, :, None] * dpu[:, None, :]).reshape(npts, -1)
    Dv = (dpv[:, :, None] * pu[:, None, :]).reshape(npts, -1)
    return P, Du, Dv
