"""Media, formulation and excitation (drop-in for chebscat.kernels, kernels.py:31-166
and 334-349).  Host-side only: the integrands themselves run on the GPU
(csrc/physics.cuh)."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
from scipy.constants import epsilon_0, mu_0, speed_of_light

MFIE_PEC = "mfie_pec"
MULLER = "muller"


@dataclass(frozen=True)
class Medium:
    eps: complex
    mu: complex
    omega: float

    @property
    def k(self) -> complex:
        k = complex(self.omega * np.sqrt(complex(self.eps) * complex(self.mu)))
        return -k if k.imag > 0 else k

    @property
    def eta(self) -> complex:
        return complex(np.sqrt(complex(self.mu) / complex(self.eps)))

    @staticmethod
    def from_relative(eps_r, mu_r, wavelength) -> "Medium":
        return Medium(eps_r * epsilon_0, mu_r * mu_0, 2.0 * np.pi * speed_of_light / wavelength)


@dataclass(frozen=True)
class FormulationSpec:
    kind: str
    outer: Medium
    inner: Optional[Medium] = None

    def __post_init__(self):
        if self.kind not in (MFIE_PEC, MULLER):
            raise ValueError(f"unknown formulation {self.kind!r}")
        if self.kind == MULLER and self.inner is None:
            raise ValueError("Muller formulation requires an inner medium")

    @property
    def n_components(self) -> int:
        return 2 if self.kind == MFIE_PEC else 4

    def scales(self):
        """Per-component equilibration (solver.py:107-117)."""
        if self.kind == MFIE_PEC:
            return np.ones(2, complex), np.ones(2, complex)
        e1, m1, z1 = self.outer.eps, self.outer.mu, self.outer.eta
        return (np.array([1 / e1, 1 / e1, z1 / m1, z1 / m1], complex),
                np.array([1 / z1, 1 / z1, 1.0, 1.0], complex))


@dataclass(frozen=True)
class PlaneWave:
    direction: np.ndarray
    polarization: np.ndarray
    amplitude: float = 1.0

    def __post_init__(self):
        d = np.asarray(self.direction, float)
        p = np.asarray(self.polarization, float)
        d = d / np.linalg.norm(d)
        p = p / np.linalg.norm(p)
        if abs(d @ p) > 1e-12:
            raise ValueError("plane-wave polarization must be orthogonal to travel")
        object.__setattr__(self, "direction", d)
        object.__setattr__(self, "polarization", p)


@dataclass(frozen=True)
class Dipole:
    """Infinitesimal electric dipole with moment p (C m) (kernels.py:126-135)."""
    position: np.ndarray
    moment: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "position", np.asarray(self.position, float))
        object.__setattr__(self, "moment", np.asarray(self.moment, float))


def incident_fields(exc, medium: Medium, points: np.ndarray):
    """(E, H) of the excitation at the points, (n, 3) each (kernels.py:141-166)."""
    pts = np.atleast_2d(np.asarray(points, float))
    k = medium.k
    if isinstance(exc, PlaneWave):
        E = exc.amplitude * np.exp(-1j * k * (pts @ exc.direction))[:, None] * exc.polarization[None, :]
        return E, np.cross(exc.direction, E) / medium.eta
    if isinstance(exc, Dipole):
        from .errors import SingularPoint
        rel = pts - exc.position
        R = np.linalg.norm(rel, axis=1)
        if np.any(R < 1e-14):
            raise SingularPoint("field point coincides with the dipole")
        rhat = rel / R[:, None]
        ekr = np.exp(-1j * k * R)
        rxp = np.cross(rhat, exc.moment)
        H = (-1j * medium.omega) * ((1 + 1j * k * R) * ekr / (4 * np.pi * R * R))[:, None] * rxp
        rad = 3.0 * rhat * (rhat @ exc.moment)[:, None] - exc.moment[None, :]
        E = (ekr / (4 * np.pi * medium.eps))[:, None] * (
            (k * k / R)[:, None] * np.cross(rxp, rhat) + (1.0 / R ** 3 + 1j * k / R ** 2)[:, None] * rad)
        return E, H
    raise TypeError(f"unknown excitation {type(exc)!r}")


def rhs_rows(spec: FormulationSpec, exc, pos, a_u, a_v) -> np.ndarray:
    """Tested incident rows per point, (n, C) (kernels.py:334-349)."""
    m = spec.outer
    E, H = incident_fields(exc, m, pos)
    hu = -np.sum(a_v * H, axis=1)
    hv = np.sum(a_u * H, axis=1)
    if spec.kind == MFIE_PEC:
        return np.stack([hu, hv], axis=1)
    eu = -np.sum(a_v * E, axis=1)
    ev = np.sum(a_u * E, axis=1)
    return np.stack([m.eps * eu, m.eps * ev, m.mu * hu, m.mu * hv], axis=1)
