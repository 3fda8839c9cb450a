"""Config builders and end-to-end oracle pipelines (restates solver.py:132-203).

Configs follow BASELINE.json / SURVEY.md section 8(d); lambda = 1 m.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from . import hcompress as hc
from . import hfactor as hf
from . import nearfield as nf
from . import physics as ph
from . import surface as sf


@dataclass
class Case:
    surfs: list
    form: ph.Form
    direction: tuple
    polarization: tuple
    aca_tol: float
    eta: float
    n_leaf: int
    tau: float = 1.0
    grading: int = 3

    def disc(self):
        return nf.Discretisation(self.surfs, self.form, self.tau, None, self.grading)


def case(cfg: int) -> Case:
    vac = ph.Medium.relative(1.0, 1.0, 1.0)
    mf = ph.Form("mfie", vac)
    if cfg == 1:
        return Case(sf.sphere_mesh(0.5, 2, (6, 6)), mf, (0, 0, 1), (1, 0, 0), 1e-6, 1.0, 128)
    if cfg == 2:
        return Case(sf.sphere_mesh(2.0, 4, (8, 8)), mf, (0, 0, 1), (1, 0, 0), 1e-4, 1.0, 256)
    if cfg == 3:
        mu = ph.Form("muller", vac, ph.Medium.relative(16.0, 1.0, 1.0))
        return Case(sf.sphere_mesh(1.0, 4, (8, 8)), mu, (0, 0, 1), (1, 0, 0), 1e-5, 1.0, 256)
    if cfg == 4:
        from paper_2408_17116_b200 import configs
        from paper_2408_17116_b200.geometry import star_coefficients
        coef, rng = star_coefficients(configs.STAR_SEED)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        p = rng.standard_normal(3)
        p -= (p @ d) * d
        p /= np.linalg.norm(p)
        return Case(sf.star_mesh(2.5, 8, (8, 8), coef), mf, tuple(d), tuple(p), 1e-4, 1.0, 256)
    if cfg == 5:
        return Case(sf.sphere_mesh(8.0, 20, (8, 8)), mf, (0, 0, 1), (1, 0, 0), 1e-4, 1.0, 512)
    raise ValueError(f"config {cfg} not available in the oracle")


def small_case(order=4, kind="mfie", eps2=4.0, aca_tol=1e-4, eta=2.0, n_leaf=64):
    """The reference test-suite's small problem (tests/test_solver.py:10-21)."""
    vac = ph.Medium.relative(1.0, 1.0, 1.0)
    form = ph.Form("mfie", vac) if kind == "mfie" else \
        ph.Form("muller", vac, ph.Medium.relative(eps2, 1.0, 1.0))
    return Case(sf.sphere_mesh(0.5, 1, (order, order)), form, (0, 0, 1), (1, 0, 0),
                aca_tol, eta, n_leaf)


def build_hmatrix(cs: Case, disc=None, sample=None):
    disc = disc or cs.disc()
    gen = nf.Scaled(disc)
    t0 = time.perf_counter()
    H = hc.HMat(disc.pos, disc.C, cs.n_leaf, cs.eta)
    t1 = time.perf_counter()
    H.fill(gen, cs.aca_tol, sample=sample)
    t2 = time.perf_counter()
    return H, disc, gen, {"tree_s": t1 - t0, "fill_s": t2 - t1}


def solve_direct(cs: Case):
    H, disc, gen, t = build_hmatrix(cs)
    b = disc.rhs(cs.direction, cs.polarization) * gen.row_scale
    t0 = time.perf_counter()
    F = hf.Factors(H, cs.aca_tol)
    t["factor_s"] = time.perf_counter() - t0
    x = F.solve(b) * gen.col_scale
    res = np.linalg.norm(H.matvec(x / gen.col_scale) - b) / np.linalg.norm(b)
    return x, res, H, t


def solve_dense(cs: Case, disc=None):
    disc = disc or cs.disc()
    A = disc.dense()
    b = disc.rhs(cs.direction, cs.polarization)
    x = sla.lu_solve(sla.lu_factor(A), b)
    return x, A, b
