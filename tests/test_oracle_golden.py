"""Pin the CPU oracle (oracle/) against golden vectors produced by running the
reference itself (tests/golden/make_golden.py).  No GPU needed."""

import numpy as np
import pytest

from oracle import hcompress as hc
from oracle import hfactor as hf
from oracle import nearfield as nf
from oracle import pipeline as pl
from oracle import spectral as sp
from oracle import surface as sf
from gold import golden


def test_spectral_tables():
    g = golden("spectral.npz")
    for n in (4, 5, 6, 8, 16):
        x, w = sp.fejer(n)
        assert np.array_equal(x, g[f"fejer_x_{n}"])
        assert np.abs(w - g[f"fejer_w_{n}"]).max() < 1e-15
        assert np.abs(sp.node_diff(n) - g[f"dnode_{n}"]).max() < 1e-12
    P, Du, Dv = sp.cardinal(6, 8, g["card_u"], g["card_v"])
    assert np.abs(P - g["card_P"]).max() < 1e-14
    assert np.abs(Du - g["card_dU"]).max() < 1e-12
    assert np.abs(Dv - g["card_dV"]).max() < 1e-12
    assert np.array_equal(sp.clenshaw2d(g["clen_c"], g["card_u"], g["card_v"]), g["clen_val"])


def test_geometry_frames():
    g = golden("geometry.npz")
    s = pl.case(1).surfs[5]
    assert np.array_equal(s.samples, g["samples"])
    pos, au, av, sg = s.frames(g["u"], g["v"])
    for a, b in ((pos, "pos"), (au, "au"), (av, "av"), (sg, "sg")):
        assert np.abs(a - g[b]).max() < 1e-15
    for a, b in zip(s.hessian_parts(g["u"], g["v"]), ("ruu", "ruv", "rvv")):
        assert np.abs(a - g[b]).max() < 1e-13
    c = sf.Surf(s.samples.copy())
    pos, au, av, sg = c.frames(g["u"], g["v"])
    assert np.abs(pos - g["cheb_pos"]).max() < 1e-14
    assert np.abs(au - g["cheb_au"]).max() < 1e-13
    assert abs(s.diameter() - float(g["diam"])) == 0.0


@pytest.fixture(scope="module")
def cfg1_disc():
    d = pl.case(1).disc()
    d.classify_all()
    return d


def _table(d):
    keys = sorted(d.cls)
    rec = np.array([(p, q, *d.cls[(p, q)]) for p, q in keys], dtype=float)
    return rec


def test_cfg1_classification_matches_reference(cfg1_disc):
    g = golden("cfg1_class.npz")
    rec = _table(cfg1_disc)
    assert rec.shape[0] == g["point"].size
    assert np.array_equal(rec[:, 0], g["point"]) and np.array_equal(rec[:, 1], g["patch"])
    assert np.array_equal(rec[:, 2], g["tag"])
    assert np.array_equal(rec[:, 5], g["ok"])
    assert np.abs(rec[:, 3] - g["u"]).max() < 1e-12
    assert np.abs(rec[:, 4] - g["v"]).max() < 1e-12
    assert cfg1_disc.fallbacks == int(g["fallbacks"])


def test_cfg1_pair_blocks(cfg1_disc):
    g = golden("cfg1_pairs.npz")
    for (p, q), ref in zip(g["keys"], g["blocks"]):
        got = cfg1_disc.pair_block(int(p), int(q))
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_cfg1_dense_entries(cfg1_disc):
    g = golden("cfg1_entries.npz")
    got = np.array([cfg1_disc.entry(i, j) for i, j in zip(g["i"], g["j"])])
    ref = g["val"]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_muller_pair_blocks():
    cs = pl.small_case(order=5, kind="muller", eps2=4.0, aca_tol=1e-5)
    d = cs.disc()
    d.classify_all()
    gc = golden("muller_class.npz")
    rec = _table(d)
    assert np.array_equal(rec[:, 2], gc["tag"])
    g = golden("muller_pairs.npz")
    for (p, q), ref in zip(g["keys"], g["blocks"]):
        got = d.pair_block(int(p), int(q))
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_tree_matches_reference(cfg1_disc):
    g = golden("cfg1_solve.npz")
    H = hc.HMat(cfg1_disc.pos, 2, 128, 1.0)
    assert np.array_equal(H.dof_perm, g["dof_perm"])
    lv = [(b.r.lo, b.r.hi, b.c.lo, b.c.hi, 1 if b.kind == "R" else 0) for b in hc.leaves(H.root)]
    assert np.array_equal(np.array(lv), g["leaves"])


def test_aca_and_truncation_kat():
    g = golden("aca.npz")
    M = g["M"]
    U, V = hc.aca(lambda i: M[i].copy(), lambda j: M[:, j].copy(), 60, 50, 1e-4)
    assert U.shape[1] == int(g["rank"])
    assert np.abs(U @ V - g["UV"]).max() < 1e-12 * np.abs(M).max()


def test_small_direct_and_dense_match_reference():
    g = golden("small_solve.npz")
    cs = pl.small_case(order=4)
    x, res, H, _ = pl.solve_direct(cs)
    assert np.linalg.norm(x - g["x_direct"]) <= 1e-10 * np.linalg.norm(g["x_direct"])
    xd, A, b = pl.solve_dense(cs)
    assert np.linalg.norm(xd - g["x_dense"]) <= 1e-12 * np.linalg.norm(g["x_dense"])
    assert np.abs(b - g["rhs"]).max() < 1e-15


def test_muller_direct_matches_reference():
    g = golden("muller_solve.npz")
    cs = pl.small_case(order=5, kind="muller", eps2=4.0, aca_tol=1e-5)
    x, res, H, _ = pl.solve_direct(cs)
    assert np.linalg.norm(x - g["x_direct"]) <= 1e-9 * np.linalg.norm(g["x_direct"])


@pytest.mark.slow
def test_cfg1_direct_matches_reference():
    g = golden("cfg1_solve.npz")
    x, res, H, _ = pl.solve_direct(pl.case(1))
    assert H.demoted == int(g["demoted"])
    assert np.linalg.norm(x - g["x_direct"]) <= 1e-9 * np.linalg.norm(g["x_direct"])


@pytest.mark.parametrize("cfg", [2, 4])
def test_oracle_classification_matches_reference_at_scale(cfg):
    """Oracle pinned on BASELINE configs 2 and 4 (config 4: the star chart) against
    the reference's full classification tables (tests/golden/make_golden_big.py)."""
    g = golden(f"cfg{cfg}_class.npz")
    d = pl.case(cfg).disc()
    d.classify_all()
    rec = _table(d)
    assert rec.shape[0] == g["point"].size
    assert np.array_equal(rec[:, 0], g["point"]) and np.array_equal(rec[:, 1], g["patch"])
    assert np.array_equal(rec[:, 2], g["tag"])
    assert np.array_equal(rec[:, 5], g["ok"])
    assert np.abs(rec[:, 3] - g["u"]).max() < 1e-12
    assert d.fallbacks == int(g["fallbacks"])


def test_oracle_sampled_leaves_match_reference_cfg2():
    g = golden("cfg2_class.npz")
    cs = pl.case(2)
    d = cs.disc()
    gen = nf.Scaled(d)
    worst = 0.0
    for rows, cols, ref in list(zip(g["leaf_rows"], g["leaf_cols"], g["leaf_vals"]))[::8]:
        got = gen.block(rows, cols)
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst <= 1e-12, worst
