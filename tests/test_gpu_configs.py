"""GPU parity on BASELINE configs 2-5 against the REFERENCE run on the same inputs
(fixtures: tests/golden/make_golden_big.py, which runs chebscat itself).

Bars (BASELINE.json north_star):
* classification: tags and Newton-convergence flags exact, (u*, v*) to 1e-11,
  fallback count exact (config 5: the 12 reference-classified patch columns);
* fill: 64 seeded leaves per config (32 dense, 32 admissible), a seeded sub-block
  of each through EquilibratedGenerator.block -- max |dA| / max |A| <= 1e-10 per leaf;
* solution: relative L2 distance to the reference's solve_direct x <= 10 * aca_tol;
* RCS (phi = 0 cut, 181 angles): <= 0.05 dB where sigma > 1e-3 max sigma.
"""

import os

import numpy as np
import pytest

from gold import GOLDEN, golden

pytestmark = pytest.mark.gpu

FILL_TOL = 1e-10
RCS_DB = 0.05
THETA = np.linspace(0.0, 180.0, 181)
_GENS = {}


def _gen(cfg):
    from paper_2408_17116_b200 import configs
    if cfg not in _GENS:
        _GENS.clear()                 # one config's device state at a time
        prob = configs.problem(cfg)
        _GENS[cfg] = (prob, prob.generator())
    return _GENS[cfg]


def _have(name):
    return os.path.exists(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_classification_matches_reference(cfg):
    g = golden(f"cfg{cfg}_class.npz")
    prob, gen = _gen(cfg)
    c = gen.classification()
    keep = np.isin(c["patch"], g["pids"])
    order = np.lexsort((c["patch"][keep], c["point"][keep]))
    c = {k: v[keep][order] for k, v in c.items()}
    assert c["point"].size == g["point"].size
    assert np.array_equal(c["point"], g["point"]) and np.array_equal(c["patch"], g["patch"])
    assert np.array_equal(c["tag"], g["tag"])
    assert np.array_equal(c["ok"], g["ok"])
    assert np.abs(c["u"] - g["u"]).max() < 1e-11
    assert np.abs(c["v"] - g["v"]).max() < 1e-11
    if g["pids"].size == int(g["npatch"]):
        assert gen.newton_fallbacks == int(g["fallbacks"])
    else:
        assert int(np.sum(c["ok"] == 0)) == int(g["fallbacks"])


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_sampled_leaves_match_reference(cfg):
    from paper_2408_17116_b200.assembly import ScaledView
    g = golden(f"cfg{cfg}_class.npz")
    prob, gen = _gen(cfg)
    sv = ScaledView(gen)
    worst = 0.0
    for rows, cols, ref in zip(g["leaf_rows"], g["leaf_cols"], g["leaf_vals"]):
        got = sv.block(rows, cols)
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst <= FILL_TOL, worst


def test_tree_matches_reference_on_configs():
    """dof permutation of the reference's cluster tree (configs 2-5)."""
    from paper_2408_17116_b200 import hmatrix as hm
    for cfg in (2, 4):
        g = golden(f"cfg{cfg}_class.npz")
        prob, gen = _gen(cfg)
        H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
        perm, lv = H.tree()
        assert np.array_equal(perm, g["leaf_dof_perm"])
        assert lv.shape[0] == int(g["leaf_n_leaves"])
        assert int((lv[:, 4] == 1).sum()) == int(g["leaf_n_adm"])


def _solution_parity(cfg, name):
    from paper_2408_17116_b200 import postprocess as post
    from paper_2408_17116_b200.solver import solve_direct
    g = golden(name)
    prob, gen = _gen(cfg)
    r = solve_direct(prob)
    x, xr = r.solution, g["x"]
    rel = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    assert rel <= 10 * prob.aca_tol, rel
    assert r.metrics["device"]["hlu"].get("trunc_overflow", 0) == 0
    _, db = post.rcs_cut(prob, gen, x, 0.0, THETA)
    sig_r = 10.0 ** (g["rcs_db"] / 10.0)
    mask = sig_r > 1e-3 * sig_r.max()
    d = np.abs(db - g["rcs_db"])
    assert d[mask].max() <= RCS_DB, d[mask].max()
    return rel, d


def test_cfg2_solution_and_rcs_match_reference():
    rel, d = _solution_parity(2, "cfg2_solve.npz")
    # diagnostic: the reference's own H solution is 1.68e-4 from its dense solution
    xd = golden("cfg2_dense.npz")["x"]
    from paper_2408_17116_b200.solver import solve_direct
    prob, gen = _gen(2)
    x = solve_direct(prob).solution
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) <= 10 * prob.aca_tol


@pytest.mark.skipif(not _have("cfg3_solve.npz"), reason="reference config-3 solve not generated")
def test_cfg3_solution_and_rcs_match_reference():
    _solution_parity(3, "cfg3_solve.npz")


@pytest.mark.skipif(not _have("cfg4_solve.npz"), reason="reference config-4 solve not generated")
def test_cfg4_solution_and_rcs_match_reference():
    _solution_parity(4, "cfg4_solve.npz")


def _mie_error(cfg, gen, x):
    from paper_2408_17116_b200 import postprocess as post
    g = golden(f"cfg{cfg}_mie.npz")
    npn = gen.nu * gen.nv
    idx = (g["pids"][:, None] * npn + np.arange(npn)[None, :]).ravel()
    assert np.abs(gen.pos[idx] - g["pos"]).max() < 1e-12     # same node points
    return post.current_error(gen, x, idx, g["J"], g["w"])


def test_cfg2_current_matches_mie_like_the_reference():
    """Surface current vs the reference's Mie series (mie.py:285-298): the GPU H solution is
    as accurate as the reference's own H solution (3.9e-4)."""
    from paper_2408_17116_b200.solver import solve_direct
    prob, gen = _gen(2)
    x = solve_direct(prob).solution
    ours = _mie_error(2, gen, x)
    ref = _mie_error(2, gen, golden("cfg2_solve.npz")["x"])
    assert ours <= 1e-3 and abs(ours - ref) <= 0.1 * ref, (ours, ref)


def test_clipped_temporary_rank_refactors(monkeypatch):
    """Temporary low-rank products get rank-sized capacities (csrc/hlu.cu tcap).  With the
    capacities forced far too small every product is clipped: the clipped recompressions are
    counted, the factorisation is redone with full-size temporaries, and the solution still
    matches the reference's (the reference's truncate_lowrank has no cap, hmatrix.py:412-426)."""
    from paper_2408_17116_b200.solver import solve_direct
    monkeypatch.setenv("CBIE_TMP_CAP_MULT", "0.02")
    g = golden("cfg2_solve.npz")
    prob, gen = _gen(2)
    r = solve_direct(prob)
    st = r.metrics["device"]["hlu"]
    assert st.get("cap_retries", 0) >= 1 and st.get("trunc_overflow", 0) == 0, st
    rel = np.linalg.norm(r.solution - g["x"]) / np.linalg.norm(g["x"])
    assert rel <= 10 * prob.aca_tol, rel


def test_two_source_recompression_matches_reference(monkeypatch):
    """CBIE_TWO_SOURCE=1: T + s U V^H is recompressed from its two pieces read in place
    (no materialised concatenation, output over the target).  Same solution as the
    concatenating default, within the reference bar."""
    from paper_2408_17116_b200.solver import solve_direct
    monkeypatch.setenv("CBIE_TWO_SOURCE", "1")
    g = golden("cfg2_solve.npz")
    prob, gen = _gen(2)
    r = solve_direct(prob)
    st = r.metrics["device"]["hlu"]
    assert st.get("trunc_overflow", 0) == 0 and st.get("tasks_concat", 1) < 0.6 * st.get("tasks_trunc", 0), st
    rel = np.linalg.norm(r.solution - g["x"]) / np.linalg.norm(g["x"])
    assert rel <= 10 * prob.aca_tol, rel


@pytest.mark.slow
def test_cfg3_hlu_completes_beyond_the_demotion_budget():
    """Config 3 (Mueller, eps_r = 16, tol 1e-5): 664 fill-in ranks exceed min(m, n) / 2.  The
    reference's truncate_lowrank has no cap (hmatrix.py:412-426); here the first attempt counts
    the clipped truncations and the re-factorisation with full-size capacities keeps every
    singular value, so the solve meets the residual bar instead of raising RankOverflow."""
    from paper_2408_17116_b200 import hmatrix as hm
    prob, gen = _gen(3)
    H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
    F = hm.hlu_factor(H, prob.effective_trunc_tol)
    st = F.stats()
    assert st["trunc_overflow"] == 0 and st.get("cap_boost", 1) > 1, st
    b = gen.rhs(prob.excitation) * gen.row_scale
    x = F.solve(b)
    res = np.linalg.norm(H.matvec(x) - b) / np.linalg.norm(b)
    assert res <= 100 * prob.aca_tol, res
