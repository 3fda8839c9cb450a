"""GPU parity of the fill (K1 classify, K3 near blocks, K2 entries) against the
reference golden fixtures and the CPU oracle.  Bar: dense entries to 1e-10
relative (max |dA| / max |A|, BASELINE.json north_star)."""

import numpy as np
import pytest

from gold import golden

pytestmark = pytest.mark.gpu

TOL = 1e-10


def cfg1_gen():
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.assembly import GpuGenerator
    med = ker.Medium.from_relative(1.0, 1.0, 1.0)
    spec = ker.FormulationSpec(ker.MFIE_PEC, med)
    return GpuGenerator(geo.unit_sphere_patches(0.5, 1, (6, 6)), spec)


def muller_gen():
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.assembly import GpuGenerator
    spec = ker.FormulationSpec(ker.MULLER, ker.Medium.from_relative(1.0, 1.0, 1.0),
                               ker.Medium.from_relative(4.0, 1.0, 1.0))
    return GpuGenerator(geo.unit_sphere_patches(0.5, 0, (5, 5)), spec)


@pytest.fixture(scope="module")
def gen1():
    return cfg1_gen()


def _check_class(gen, g):
    c = gen.classification()
    assert c["point"].size == g["point"].size
    assert np.array_equal(c["point"], g["point"]) and np.array_equal(c["patch"], g["patch"])
    assert np.array_equal(c["tag"], g["tag"])
    assert np.array_equal(c["ok"], g["ok"])
    assert np.abs(c["u"] - g["u"]).max() < 1e-11
    assert np.abs(c["v"] - g["v"]).max() < 1e-11
    assert gen.newton_fallbacks == int(g["fallbacks"])


def test_cfg1_classification_matches_reference(gen1):
    _check_class(gen1, golden("cfg1_class.npz"))


def test_cfg1_pair_blocks_match_reference(gen1):
    g = golden("cfg1_pairs.npz")
    worst = 0.0
    for (p, q), ref in zip(g["keys"], g["blocks"]):
        got = gen1.pair_block(int(p), int(q))
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst <= TOL, worst


def test_cfg1_entries_match_reference(gen1):
    g = golden("cfg1_entries.npz")
    A = gen1.block(np.arange(gen1.n_dofs), np.arange(gen1.n_dofs))
    got = A[g["i"], g["j"]]
    assert np.abs(got - g["val"]).max() <= TOL * np.abs(g["val"]).max()


def test_cfg1_dense_fill_matches_oracle(gen1):
    from oracle import pipeline as pl
    from paper_2408_17116_b200.assembly import assemble_dense
    A = assemble_dense(gen1)
    d = pl.case(1).disc()
    B = d.dense()
    assert np.abs(A - B).max() <= TOL * np.abs(B).max()
    # fill_block over scattered rows/cols is the same generator
    rng = np.random.default_rng(3)
    r = rng.choice(gen1.n_dofs, 50, replace=False)
    c = rng.choice(gen1.n_dofs, 70, replace=False)
    assert np.array_equal(gen1.block(r, c), A[np.ix_(r, c)])


def test_cfg1_rhs_matches_reference(gen1):
    from paper_2408_17116_b200 import kernels as ker
    b = gen1.rhs(ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0))
    g = golden("cfg1_solve.npz")
    assert np.abs(b - g["rhs"]).max() < 1e-13 * np.abs(g["rhs"]).max()


def test_muller_classification_and_pair_blocks():
    gen = muller_gen()
    _check_class(gen, golden("muller_class.npz"))
    g = golden("muller_pairs.npz")
    worst = 0.0
    for (p, q), ref in zip(g["keys"], g["blocks"]):
        got = gen.pair_block(int(p), int(q))
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst <= TOL, worst


def test_muller_dense_fill_matches_oracle():
    from oracle import pipeline as pl
    from paper_2408_17116_b200.assembly import assemble_dense
    gen = muller_gen()
    A = assemble_dense(gen)
    B = pl.small_case(order=5, kind="muller", eps2=4.0).disc().dense()
    assert np.abs(A - B).max() <= TOL * np.abs(B).max()


def test_chebyshev_sample_patches_match_oracle():
    """Chart-less patches: geometry from the Chebyshev interpolant of the samples."""
    from oracle import nearfield as nf, physics as ph, surface as sf
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.assembly import GpuGenerator, assemble_dense
    charted = geo.unit_sphere_patches(0.5, 0, (5, 5))
    plain = [geo.Patch(p.id, p.samples.copy()) for p in charted]
    spec = ker.FormulationSpec(ker.MFIE_PEC, ker.Medium.from_relative(1.0, 1.0, 1.0))
    gen = GpuGenerator(plain, spec)
    A = assemble_dense(gen)
    d = nf.Discretisation([sf.Surf(p.samples.copy()) for p in plain],
                          ph.Form("mfie", ph.Medium.relative(1.0, 1.0, 1.0)))
    B = d.dense()
    assert np.abs(A - B).max() <= TOL * np.abs(B).max()


def test_star_chart_frames_match_finite_differences():
    """Config-4 star chart on the device: positions and tangents are bit-identical
    to the host chart (geometry.star_eval, the chart the reference is run with in
    tests/golden/make_golden_big.py), tangents equal central differences."""
    from paper_2408_17116_b200 import geometry as geo, kernels as ker
    from paper_2408_17116_b200.assembly import GpuGenerator
    coef, _ = geo.star_coefficients(2408)
    patches = geo.star_patches(2.5, 0, (5, 5), coef)
    spec = ker.FormulationSpec(ker.MFIE_PEC, ker.Medium.from_relative(1.0, 1.0, 1.0))
    gen = GpuGenerator(patches, spec)
    xu = geo.fejer_nodes(5)
    uu, vv = np.tile(xu, 5), np.repeat(xu, 5)
    h = 1e-6
    for q, p in enumerate(patches):
        ch = p.chart
        sl = slice(q * 25, (q + 1) * 25)
        pos, au, av = geo.star_eval(ch.radius, ch.face, ch.u_lo, ch.u_hi, ch.v_lo, ch.v_hi,
                                    ch.tables(), uu, vv)
        assert np.array_equal(gen.pos[sl], pos)
        assert np.array_equal(gen.a_u[sl], au) and np.array_equal(gen.a_v[sl], av)
        du = (ch.positions(uu + h, vv) - ch.positions(uu - h, vv)) / (2 * h)
        dv = (ch.positions(uu, vv + h) - ch.positions(uu, vv - h)) / (2 * h)
        assert np.abs(gen.a_u[sl] - du).max() < 1e-7
        assert np.abs(gen.a_v[sl] - dv).max() < 1e-7
