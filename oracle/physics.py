"""Media, kernels and tested integrand blocks (oracle restatement of kernels.py).

e^{+j omega t} convention: outgoing waves carry e^{-jkR}, Im k <= 0.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.constants import epsilon_0, mu_0, speed_of_light


@dataclass(frozen=True)
class Medium:
    eps: complex
    mu: complex
    omega: float

    @property
    def k(self) -> complex:                         # kernels.py:39-42
        k = complex(self.omega * np.sqrt(complex(self.eps) * complex(self.mu)))
        return -k if k.imag > 0 else k

    @property
    def eta(self) -> complex:                       # kernels.py:44-46
        return complex(np.sqrt(complex(self.mu) / complex(self.eps)))

    @staticmethod
    def relative(eps_r, mu_r, wavelength):          # kernels.py:48-51
        return Medium(eps_r * epsilon_0, mu_r * mu_0,
                      2.0 * np.pi * speed_of_light / wavelength)


@dataclass(frozen=True)
class Form:
    """kind 'mfie' (C=2) or 'muller' (C=4)."""
    kind: str
    outer: Medium
    inner: Medium | None = None

    @property
    def C(self):
        return 2 if self.kind == "mfie" else 4

    def jump(self):                                 # kernels.py:85-100
        if self.kind == "mfie":
            return 0.5 * np.eye(2, dtype=complex)
        j = np.zeros((4, 4), dtype=complex)
        j[0, 2] = j[1, 3] = -(self.outer.eps + self.inner.eps) / 2.0
        j[2, 0] = j[3, 1] = (self.outer.mu + self.inner.mu) / 2.0
        return j

    def scales(self):
        """Per-component row / column equilibration (solver.py:102-117)."""
        if self.kind == "mfie":
            return np.ones(2), np.ones(2)
        e1, m1, z1 = self.outer.eps, self.outer.mu, self.outer.eta
        return (np.array([1 / e1, 1 / e1, z1 / m1, z1 / m1]),
                np.array([1 / z1, 1 / z1, 1.0, 1.0]))


def _sxc(x):
    """sin x - x cos x with the |x|<0.05 series (kernels.py:196-203)."""
    x = np.asarray(x)
    small = np.abs(x) < 0.05
    xs = np.where(small, x, 0.0)
    q = xs * xs
    ser = xs * q * (1.0 / 3.0 + q * (-1.0 / 30.0 + q * (1.0 / 840.0 - q / 45360.0)))
    return np.where(small, ser, np.sin(x) - x * np.cos(x))


def mfie_block(k, xo, auo, avo, ys, aus, avs, sgs):
    """(n, 2, 2): tested -grad G x a_c' / sqrt g'  (kernels.py:234-246)."""
    rel = xo[None, :] - ys
    R = np.linalg.norm(rel, axis=1)
    f = -(1 + 1j * k * R) * np.exp(-1j * k * R) / (4 * np.pi * R ** 3)
    g = f[:, None] * rel
    t = np.stack([-avo, auo])                       # tested rows (kernels.py:229-231)
    out = np.empty((ys.shape[0], 2, 2), dtype=complex)
    out[:, :, 0] = (-np.cross(g, aus)) @ t.T
    out[:, :, 1] = (-np.cross(g, avs)) @ t.T
    return out / sgs[:, None, None]


def muller_fields(form: Form, xo, auo, avo, ys, aus, avs, sgs):
    """(T6 (n,6,2), TdG (n,2)) compact Muller generators (kernels.py:249-287)."""
    m1, m2 = form.outer, form.inner
    k1, k2, w = m1.k, m2.k, m1.omega
    rel = xo[None, :] - ys
    R = np.linalg.norm(rel, axis=1)
    G2 = np.exp(-1j * k2 * R) / (4 * np.pi * R)
    s = 0.5 * (k1 + k2)
    d = 0.5 * (k1 - k2)
    Gd = np.exp(-1j * s * R) * (-2j) * np.sin(d * R) / (4 * np.pi * R)
    g2 = (-(1 + 1j * k2 * R) * np.exp(-1j * k2 * R) / (4 * np.pi * R ** 3))[:, None] * rel
    gd = (2.0 * np.exp(-1j * s * R) * (1j * _sxc(d * R) - R * s * np.sin(d * R))
          / (4 * np.pi * R ** 3))[:, None] * rel
    em1, em2 = m1.eps * m1.mu, m2.eps * m2.mu
    sJ = 1j * w * (em1 * Gd + (em1 - em2) * G2)
    cM = m1.eps * gd + (m1.eps - m2.eps) * g2
    cJ = -(m1.mu * gd + (m1.mu - m2.mu) * g2)
    t = np.stack([-avo, auo])
    T6 = np.empty((ys.shape[0], 6, 2), dtype=complex)
    T6[:, 0] = (aus @ t.T) * sJ[:, None]
    T6[:, 1] = (avs @ t.T) * sJ[:, None]
    T6[:, 2] = np.cross(cM, aus) @ t.T
    T6[:, 3] = np.cross(cM, avs) @ t.T
    T6[:, 4] = np.cross(cJ, aus) @ t.T
    T6[:, 5] = np.cross(cJ, avs) @ t.T
    TdG = (gd / (-1j * w)) @ t.T
    return T6 / sgs[:, None, None], TdG / sgs[:, None]


def muller_expand(T6, TdG):
    """4x4 value / derivative blocks from the compact fields (kernels.py:290-307)."""
    n = T6.shape[0]
    Bv = np.empty((n, 4, 4), dtype=complex)
    Bd = np.zeros((n, 4, 4), dtype=complex)
    for c, g in enumerate((0, 1, 2, 3)):
        Bv[:, 0:2, c] = T6[:, g]
    for c, g in enumerate((4, 5, 0, 1)):
        Bv[:, 2:4, c] = T6[:, g]
    for c in range(4):
        Bd[:, (0, 1) if c < 2 else (2, 3), c] = TdG
    return Bv, Bd


def plane_wave_rows(form: Form, direction, polarization, amplitude, pos, au, av):
    """Tested incident rows per point (kernels.py:141-149, 334-349)."""
    d = np.asarray(direction, float)
    d = d / np.linalg.norm(d)
    p = np.asarray(polarization, float)
    p = p / np.linalg.norm(p)
    m = form.outer
    ph = np.exp(-1j * m.k * (pos @ d))
    E = amplitude * ph[:, None] * p[None, :]
    H = np.cross(d, E) / m.eta
    hu = -np.sum(av * H, axis=1)
    hv = np.sum(au * H, axis=1)
    if form.C == 2:
        return np.stack([hu, hv], 1)
    eu = -np.sum(av * E, axis=1)
    ev = np.sum(au * E, axis=1)
    return np.stack([m.eps * eu, m.eps * ev, m.mu * hu, m.mu * hv], 1)
