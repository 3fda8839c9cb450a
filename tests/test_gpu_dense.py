"""Dense path solve_dense (solver.py:178-203) on the device: fill, LU with partial
pivoting and solve all in HBM (cbie_dense_solve), against the reference's dense
solutions (tests/golden: cfg1_solve.npz x_dense, cfg2_dense.npz x)."""

import numpy as np
import pytest

from gold import golden

pytestmark = pytest.mark.gpu


def test_cfg1_dense_solution_matches_reference():
    from paper_2408_17116_b200 import configs
    from paper_2408_17116_b200.solver import solve_dense
    r = solve_dense(configs.problem(1))
    xr = golden("cfg1_solve.npz")["x_dense"]
    assert np.linalg.norm(r.solution - xr) <= 1e-12 * np.linalg.norm(xr)
    assert r.residual < 1e-12


def test_cfg2_dense_solution_matches_reference():
    from paper_2408_17116_b200 import configs
    from paper_2408_17116_b200.solver import solve_dense
    r = solve_dense(configs.problem(2))
    g = golden("cfg2_dense.npz")
    assert np.linalg.norm(r.solution - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
    assert r.residual < 1e-12


def test_dense_lu_factors_match_lapack():
    """Packed L\\U and interchanges equal scipy's lu_factor of the same matrix."""
    import ctypes as ct
    import scipy.linalg as sla
    from paper_2408_17116_b200 import _ffi, geometry as geo, kernels as ker
    from paper_2408_17116_b200.assembly import GpuGenerator, assemble_dense
    spec = ker.FormulationSpec(ker.MFIE_PEC, ker.Medium.from_relative(1.0, 1.0, 1.0))
    gen = GpuGenerator(geo.unit_sphere_patches(0.5, 0, (5, 5)), spec)
    A = assemble_dense(gen)
    N = A.shape[0]
    b = np.ascontiguousarray(np.arange(2 * N, dtype=complex).reshape(N, 2) + 1j)
    x = np.empty_like(b)
    lu = np.empty((N, N), complex)
    piv = np.empty(N, np.int32)
    res = ct.c_double()
    gen.dev.check(gen.dev.lib.cbie_dense_solve(gen.dev.h, 10 ** 9, _ffi.ptr(b), 2, _ffi.ptr(x), ct.byref(res),
                                               _ffi.ptr(lu), _ffi.ptr(piv)))
    lu_r, piv_r = sla.lu_factor(A)
    assert np.array_equal(piv, piv_r)
    assert np.abs(lu - lu_r).max() <= 1e-13 * np.abs(lu_r).max()
    assert np.abs(x - sla.lu_solve((lu_r, piv_r), b)).max() <= 1e-12 * np.abs(x).max()
    assert res.value < 1e-13
