"""Far-field radiation sums on the device (cbie_far_field_sums, csrc/farfield.cu)
against the reference's dense phase-matrix products (postprocess.py:193-212)
restated in numpy, for MFIE (4 tables) and Muller (8 tables)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gen(kind):
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.solver import Problem
    vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
    pw = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
    if kind == "mfie":
        prob = Problem(geo.unit_sphere_patches(0.5, 1, (6, 6)), ker.FormulationSpec(ker.MFIE_PEC, vac), pw)
    else:
        spec = ker.FormulationSpec(ker.MULLER, vac, ker.Medium.from_relative(4.0, 1.0, 1.0))
        prob = Problem(geo.unit_sphere_patches(0.5, 0, (5, 5)), spec, pw)
    return prob, prob.generator()


@pytest.mark.parametrize("kind", ["mfie", "muller"])
def test_far_field_sums_match_phase_matrix(kind):
    from paper_2408_17116_b200 import postprocess as post
    prob, gen = _gen(kind)
    rng = np.random.default_rng(7)
    x = rng.standard_normal(gen.n_dofs) + 1j * rng.standard_normal(gen.n_dofs)
    theta = np.deg2rad(np.linspace(0.0, 180.0, 37))
    phi = np.deg2rad(np.linspace(0.0, 350.0, 37))
    F, rhat = post.far_field(prob, gen, x, theta, phi)
    # numpy restatement of postprocess.py:201-212 on the same tables
    med = prob.spec.outer
    k, omega = med.k, med.omega
    pos, tabs = post.radiation_tables(gen, x)
    phase = np.exp(1j * k * (rhat @ pos.T))
    wJ, wdJ = tabs[0]
    Fr = -(1.0 / (4 * np.pi)) * (1j * omega * med.mu * (phase @ wJ)
                                 + (k / (omega * med.eps)) * rhat * (phase @ wdJ)[:, None])
    if len(tabs) > 1:
        Fr = Fr + (1.0 / (4 * np.pi)) * 1j * k * np.cross(rhat, phase @ tabs[1][0])
    Fr = Fr - rhat * np.sum(Fr * rhat, axis=1)[:, None]
    assert np.abs(F - Fr).max() <= 1e-11 * np.abs(Fr).max()


def test_far_field_refuses_empty_table_count():
    prob, gen = _gen("mfie")
    out = np.empty((1, 9), complex)
    rh = np.zeros((1, 3))
    tab = np.zeros((gen.n_points, 9), complex)
    from paper_2408_17116_b200 import _ffi
    rc = gen.dev.lib.cbie_far_field_sums(gen.dev.h, _ffi.ptr(tab), 9, _ffi.ptr(rh), 1, 1.0, _ffi.ptr(out))
    assert rc != 0
