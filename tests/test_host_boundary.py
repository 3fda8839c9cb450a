"""Host side of the drop-in boundary (no GPU): the config-4 star chart tables, the
reference-object adapter (solver.from_reference) and the Dipole excitation rows."""

import os

import numpy as np
import pytest


def test_star_tables_reproduce_real_sh_and_tangents():
    from paper_2408_17116_b200 import geometry as geo
    coef, _ = geo.star_coefficients(2408)
    T = geo.star_tables(coef).reshape(4, 35)
    rng = np.random.default_rng(1)
    v = rng.standard_normal((200, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    px = [np.ones(200)] + [v[:, 0] ** k for k in range(1, 5)]
    py = [np.ones(200)] + [v[:, 1] ** k for k in range(1, 5)]
    pz = [np.ones(200)] + [v[:, 2] ** k for k in range(1, 5)]
    assert np.abs(geo._star_poly(T[0], px, py, pz) - geo.real_sh(v) @ coef).max() < 1e-14
    ch = geo.star_patches(2.5, 1, (8, 8), coef)[9].chart
    u = np.linspace(-0.9, 0.9, 7)
    w = 0.3 * u[::-1]
    h = 1e-6
    _, au, av = geo.star_eval(ch.radius, ch.face, ch.u_lo, ch.u_hi, ch.v_lo, ch.v_hi, ch.tables(), u, w)
    pu = (ch.positions(u + h, w) - ch.positions(u - h, w)) / (2 * h)
    pv = (ch.positions(u, w + h) - ch.positions(u, w - h)) / (2 * h)
    assert np.abs(pu - au).max() < 1e-8 and np.abs(pv - av).max() < 1e-8
    # deviation normalised to 0.2 (BASELINE config 4)
    assert np.max(np.linalg.norm(ch.positions(u, w), axis=1)) <= 2.5 * 1.2 + 1e-12


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_from_reference_takes_reference_objects_unchanged():
    import sys
    sys.path.insert(0, REF)
    try:
        from chebscat import geometry as rgeo, kernels as rker, solver as rsol
    finally:
        sys.path.remove(REF)
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.solver import from_reference
    rp = rgeo.unit_sphere_patches(0.5, 1, (6, 6))
    rp[3] = rgeo.Patch(3, rp[3].samples.copy())          # one chart-less patch
    spec = rker.FormulationSpec(rker.MULLER, rker.Medium.from_relative(1.0, 1.0, 1.0),
                                rker.Medium.from_relative(4.0, 1.0, 1.0))
    prob = rsol.Problem(rp, spec, rker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0), aca_tol=1e-5,
                        eta=1.0, n_leaf=128)
    p = from_reference(prob)
    mine = geo.unit_sphere_patches(0.5, 1, (6, 6))
    for a, b in zip(p.patches, mine):
        assert np.array_equal(a.samples, b.samples)
    smp, kind, par, star, coef = geo.device_arrays(p.patches)
    _, kind2, par2, _, _ = geo.device_arrays(mine)
    assert kind[3] == geo.CHART_SAMPLES and np.array_equal(np.delete(par, 3, 0), np.delete(par2, 3, 0))
    assert p.spec.kind == ker.MULLER and p.spec.inner.eps == spec.inner.eps
    assert (p.aca_tol, p.eta, p.n_leaf) == (1e-5, 1.0, 128)
    # the host RHS rows equal the reference's for plane waves and dipoles
    frames = rp[0].node_frames()
    for exc, mexc in ((prob.excitation, p.excitation),
                      (rker.Dipole([0.1, 0.0, 2.0], [0.0, 1.0, 0.5]),
                       ker.Dipole([0.1, 0.0, 2.0], [0.0, 1.0, 0.5]))):
        ref = rker.rhs_rows(spec, exc, frames)
        got = ker.rhs_rows(p.spec, mexc, frames.position, frames.a_u, frames.a_v)
        assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()
