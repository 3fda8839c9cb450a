"""The five BASELINE.json configurations; lambda = 1 m."""

from __future__ import annotations

import numpy as np

from . import geometry as geo
from . import kernels as ker
from .solver import Problem

STAR_SEED = 2408


def problem(cfg: int) -> Problem:
    vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
    mfie = ker.FormulationSpec(ker.MFIE_PEC, vac)
    z = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
    if cfg == 1:
        return Problem(geo.unit_sphere_patches(0.5, 1, (6, 6)), mfie, z,
                       aca_tol=1e-6, eta=1.0, n_leaf=128)
    if cfg == 2:
        return Problem(geo.unit_sphere_patches(2.0, 2, (8, 8)), mfie, z,
                       aca_tol=1e-4, eta=1.0, n_leaf=256)
    if cfg == 3:
        spec = ker.FormulationSpec(ker.MULLER, vac, ker.Medium.from_relative(16.0, 1.0, 1.0))
        return Problem(geo.unit_sphere_patches(1.0, 2, (8, 8)), spec, z,
                       aca_tol=1e-5, eta=1.0, n_leaf=256)
    if cfg == 4:
        coef, rng = geo.star_coefficients(STAR_SEED)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        p = rng.standard_normal(3)
        p -= (p @ d) * d
        p /= np.linalg.norm(p)
        return Problem(geo.star_patches(2.5, 3, (8, 8), coef), mfie, ker.PlaneWave(d, p, 1.0),
                       aca_tol=1e-4, eta=1.0, n_leaf=256)
    if cfg == 5:
        return Problem(geo.sphere_patches(8.0, np.linspace(-1.0, 1.0, 21), (8, 8)), mfie, z,
                       aca_tol=1e-4, eta=1.0, n_leaf=512)
    raise ValueError(f"unknown config {cfg}")
