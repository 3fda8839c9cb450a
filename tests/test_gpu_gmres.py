"""Device GMRES on the H-matvec (cbie_gmres; solver.gmres / solve_gmres,
solver.py:206-307) against the H-LU direct solution of the same H-matrix and
against the reference's golden solution (config 1)."""

import numpy as np
import pytest

from gold import golden

pytestmark = pytest.mark.gpu


def _cfg1(**kw):
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.solver import Problem
    vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
    return Problem(geo.unit_sphere_patches(0.5, 1, (6, 6)), ker.FormulationSpec(ker.MFIE_PEC, vac),
                   ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0), aca_tol=1e-6, eta=1.0, n_leaf=128, **kw)


def test_gmres_converges_to_direct_solution():
    from paper_2408_17116_b200.solver import solve_direct, solve_gmres
    prob = _cfg1(gmres_tol=1e-8)
    rg = solve_gmres(prob)
    rd = solve_direct(prob)
    assert rg.converged and 0 < rg.iterations < 200
    assert rg.residual <= 1e-8
    assert np.linalg.norm(rg.solution - rd.solution) / np.linalg.norm(rd.solution) <= 1e-6
    g = golden("cfg1_solve.npz")
    assert np.linalg.norm(rg.solution - g["x_direct"]) / np.linalg.norm(g["x_direct"]) <= 10 * prob.aca_tol


def test_gmres_restart_and_iteration_cap():
    from paper_2408_17116_b200.solver import solve_gmres
    prob = _cfg1(gmres_tol=1e-10)
    r = solve_gmres(prob, restart=5, max_iters=12)
    assert r.iterations == 12 and not r.converged and r.residual > 1e-10
    r2 = solve_gmres(prob, restart=5, max_iters=400)
    assert r2.converged and r2.residual <= 1e-10


def test_small_problem_iterates_on_the_dense_operator():
    """N <= 600: the reference's solve_gmres uses the dense equilibrated matrix
    (solver.py:278-287); here one dense leaf covers the matrix and the metrics say so."""
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.solver import Problem, solve_gmres
    vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
    prob = Problem(geo.unit_sphere_patches(0.5, 0, (4, 4)), ker.FormulationSpec(ker.MFIE_PEC, vac),
                   ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0), gmres_tol=1e-10)
    r = solve_gmres(prob)
    assert r.metrics["operator"] == "dense" and r.converged
    assert r.metrics["compression_rate"] <= 1e-12          # nothing compressed: one dense leaf
    g = golden("small_solve.npz")
    assert np.linalg.norm(r.solution - g["x_dense"]) / np.linalg.norm(g["x_dense"]) <= 1e-8
