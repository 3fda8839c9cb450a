"""Golden fixtures for BASELINE configs 2-5, produced by running the REFERENCE.

Build container only (the reference does not exist on the GPU box).  Each job is
one invocation so the long ones can run side by side, one core each:

    PYTHONPATH=/root/reference/pkg/src:. PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden_big.py cfg2_class      # classification table + sampled leaves
        python tests/golden/make_golden_big.py cfg2_solve      # solve_direct x, RCS, timings (1 thread)
        python tests/golden/make_golden_big.py cfg2_dense      # solve_dense x, RCS (diagnostic)
        python tests/golden/make_golden_big.py cfg3_class | cfg3_solve
        python tests/golden/make_golden_big.py cfg4_class | cfg4_solve
        python tests/golden/make_golden_big.py cfg5_leaves

Every array comes from the reference's public functions (solver.solve_direct,
solver.solve_dense, EquilibratedGenerator.block, EntryGenerator's classification
cache, postprocess.rcs_cut).  The problems are the SURVEY.md section 8(d)
configurations; configs 4 and 5 are built from reference ``Chart`` objects:
config 4 with ``RefStarFace`` below (the star chart of
paper_2408_17116_b200/geometry.py restated over the reference's Chart interface,
same floating-point operation order as the device chart so positions and
tangents agree bit for bit), config 5 with the reference's own CubeSphereFace on
a 20 x 20 face split (SURVEY.md section 7 hard part 7).

Sampled leaves: for 32 seeded dense and 32 seeded admissible leaves of the
reference's block tree, a seeded 24 x 24 sub-block (rows/cols in original dof
numbering) of the equilibrated system via ``EquilibratedGenerator.block``
(solver.py:127-129) -- the exact entries every leaf of the H-matrix is built
from.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from chebscat import assembly as asm           # noqa: E402
from chebscat import chebyshev as cheb         # noqa: E402
from chebscat import geometry as rgeo          # noqa: E402
from chebscat import hmatrix as hm             # noqa: E402
from chebscat import kernels as ker            # noqa: E402
from chebscat import postprocess as post       # noqa: E402
from chebscat import quadrature as quad        # noqa: E402
from chebscat import solver as rsolver         # noqa: E402

THETA = np.linspace(0.0, 180.0, 181)
STAR_SEED = 2408


def save(name, **arrs):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)", flush=True)


# --------------------------------------------------------------------------- star chart
class RefStarFace(rgeo.CubeSphereFace):
    """Config-4 chart over the reference's Chart interface (geometry.py:38-97).

    r(xhat) = a (1 + sum_i c_i Y_i(xhat)) xhat on the cube -> sphere direction map;
    c already carries the 0.2 / max|sum c Y| normalisation.  Operation order
    follows csrc/geometry.cuh star_chart (explicitly rounded there), elementwise
    here, so both round identically."""

    def __init__(self, a, face, u_lo, u_hi, v_lo, v_hi, coef):
        from paper_2408_17116_b200 import geometry as g
        super().__init__(a, face, u_lo, u_hi, v_lo, v_hi)
        self.coef = np.asarray(coef, float)
        self.tables = g.star_tables(self.coef)

    def _eval(self, u, v):
        from paper_2408_17116_b200 import geometry as g
        return g.star_eval(self.radius, self.face, self.u_lo, self.u_hi, self.v_lo, self.v_hi,
                           self.tables, np.asarray(u, float).ravel(),
                           np.asarray(v, float).ravel())

    def positions(self, u, v):
        return self._eval(u, v)[0]

    def derivatives(self, u, v):
        _, au, av = self._eval(u, v)
        return au, av


def _patches_from_charts(charts, order):
    nu, nv = order
    un = cheb.fejer1(nu).nodes
    vn = cheb.fejer1(nv).nodes
    V, U = np.meshgrid(vn, un, indexing="ij")
    out = []
    for pid, ch in enumerate(charts):
        pos = ch.positions(U.ravel(), V.ravel())
        out.append(rgeo.Patch(pid, pos.reshape(nv, nu, 3).transpose(1, 0, 2).copy(), chart=ch))
    return out


def ref_problem(cfg: int, workers: int = 1):
    vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
    mfie = ker.FormulationSpec(ker.MFIE_PEC, vac)
    z = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
    if cfg == 2:
        return rsolver.Problem(rgeo.unit_sphere_patches(2.0, 2, (8, 8)), mfie, z,
                               aca_tol=1e-4, eta=1.0, n_leaf=256, workers=workers)
    if cfg == 3:
        spec = ker.FormulationSpec(ker.MULLER, vac, ker.Medium.from_relative(16.0, 1.0, 1.0))
        return rsolver.Problem(rgeo.unit_sphere_patches(1.0, 2, (8, 8)), spec, z,
                               aca_tol=1e-5, eta=1.0, n_leaf=256, workers=workers,
                               dense_cap=10 ** 9)
    if cfg == 4:
        from paper_2408_17116_b200 import geometry as g
        coef, rng = g.star_coefficients(STAR_SEED)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        p = rng.standard_normal(3)
        p -= (p @ d) * d
        p /= np.linalg.norm(p)
        e = np.linspace(-1.0, 1.0, 9)
        charts = [RefStarFace(2.5, f, e[iu], e[iu + 1], e[iv], e[iv + 1], coef)
                  for f in range(6) for iu in range(8) for iv in range(8)]
        return rsolver.Problem(_patches_from_charts(charts, (8, 8)), mfie,
                               ker.PlaneWave(d, p, 1.0), aca_tol=1e-4, eta=1.0, n_leaf=256,
                               workers=workers)
    if cfg == 5:
        e = np.linspace(-1.0, 1.0, 21)
        charts = [rgeo.CubeSphereFace(8.0, f, e[iu], e[iu + 1], e[iv], e[iv + 1])
                  for f in range(6) for iu in range(20) for iv in range(20)]
        return rsolver.Problem(_patches_from_charts(charts, (8, 8)), mfie, z,
                               aca_tol=1e-4, eta=1.0, n_leaf=512, workers=workers)
    raise ValueError(cfg)


# --------------------------------------------------------------------------- pieces
def classification(gen, pids=None):
    """Non-FAR rows of the reference's classification cache (assembly.py:106-143)."""
    P = len(gen.patches)
    pids = range(P) if pids is None else pids
    t0 = time.perf_counter()
    for pid in pids:
        gen._classify_patch_column(pid)
    sec = time.perf_counter() - t0
    rec = []
    for (pt, pid), ic in gen._class_cache.items():
        if ic.tag == quad.FAR:
            continue
        rec.append((pt, pid, 1 if ic.tag == quad.NEAR else 2, ic.uv[0], ic.uv[1],
                    1 if ic.newton_ok else 0))
    rec.sort()
    a = np.array(rec, dtype=float)
    return dict(point=a[:, 0].astype(np.int32), patch=a[:, 1].astype(np.int32),
                tag=a[:, 2].astype(np.int8), u=a[:, 3], v=a[:, 4], ok=a[:, 5].astype(np.int8),
                fallbacks=gen.newton_fallbacks, npts=gen.dofmap.n_points, npatch=P,
                pids=np.array(list(pids), np.int32), classify_s=sec)


def tree_leaves(prob, gen):
    pts = gen.dofmap.point_positions()
    tree = hm.build_cluster_tree(pts, prob.spec.n_components, prob.n_leaf)
    H = hm.build_block_tree(tree, prob.eta)
    leaves = []

    def walk(b, r, c):
        if isinstance(b, hm.HBlock):
            for i, rk in enumerate(b.rows):
                for k, ck in enumerate(b.cols):
                    walk(b.children[i][k], rk, ck)
        else:
            leaves.append((r, c, 1 if isinstance(b, hm._PendingLowRank) else 0))

    walk(H.root, tree.root, tree.root)
    return tree, leaves


def sampled_leaves(prob, gen, n_each=32, sub=24, seed=31):
    """Seeded sub-blocks of seeded leaves via EquilibratedGenerator.block."""
    scaled = rsolver.EquilibratedGenerator(gen)
    tree, leaves = tree_leaves(prob, gen)
    rng = np.random.default_rng(seed)
    pick = []
    for adm in (0, 1):
        idx = [i for i, lf in enumerate(leaves) if lf[2] == adm]
        pick += sorted(rng.choice(idx, size=min(n_each, len(idx)), replace=False).tolist())
    rows, cols, vals, meta = [], [], [], []
    t0 = time.perf_counter()
    for li in pick:
        r, c, adm = leaves[li]
        rd = tree.node_dofs(r)
        cd = tree.node_dofs(c)
        ri = np.sort(rng.choice(rd.size, size=min(sub, rd.size), replace=False))
        ci = np.sort(rng.choice(cd.size, size=min(sub, cd.size), replace=False))
        rows.append(rd[ri])
        cols.append(cd[ci])
        vals.append(scaled.block(rd[ri], cd[ci]))
        meta.append((li, adm, r.lo, r.hi, c.lo, c.hi))
    sec = time.perf_counter() - t0
    return dict(rows=np.array(rows, np.int64), cols=np.array(cols, np.int64),
                vals=np.array(vals), meta=np.array(meta, np.int64),
                n_leaves=len(leaves), n_adm=sum(lf[2] for lf in leaves),
                dof_perm=tree.dof_perm.astype(np.int64), sample_s=sec)


def solve(prob, dense=False):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        t0 = time.perf_counter()
        r = rsolver.solve_dense(prob) if dense else rsolver.solve_direct(prob)
        wall = time.perf_counter() - t0
    m = {k: v for k, v in r.metrics.items() if isinstance(v, (int, float, str))}
    m["wall_s"] = wall
    m["threads"] = "workers=%d, BLAS=1 (threadpool_limits)" % prob.workers
    cut = post.rcs_cut(prob, r.solution, 0.0, THETA)
    return dict(x=r.solution, residual=r.residual, rcs_db=cut.sigma_dbsm,
                metrics=json.dumps(m, default=str))


def mie_currents(cfg, n_patch=None, seed=41):
    """The reference's Mie-series surface current J = n x H (mie.py:285-298) at the node
    points of (a seeded subset of) the patches, with the node weights w sqrt(g) used by
    postprocess.mie_comparison (postprocess.py:275-314)."""
    from chebscat import mie
    prob = ref_problem(cfg)
    radius = {2: 2.0, 5: 8.0}[cfg]
    P = len(prob.patches)
    pids = np.arange(P) if n_patch is None else np.sort(
        np.random.default_rng(seed).choice(P, size=n_patch, replace=False))
    spec = mie.MieSpec(radius, prob.spec.outer, None, amplitude=prob.excitation.amplitude)
    J, W, pts = [], [], []
    for q in pids:
        p = prob.patches[int(q)]
        fb = p.node_frames()
        Jm, _ = mie.mie_surface_current(spec, fb.position)
        J.append(Jm)
        W.append(p.node_weights() * fb.sqrt_g)
        pts.append(fb.position)
    save(f"cfg{cfg}_mie.npz", pids=pids.astype(np.int32), J=np.concatenate(J), w=np.concatenate(W),
         pos=np.concatenate(pts), n_terms=spec.n_terms)


def thread_sweep(cfg):
    """The reference's config run under the two other thread settings of BASELINE.md 3
    (setting 1, workers=1 / BLAS=1, is cfgN_solve): workers=cores with BLAS=1, and
    workers=1 with BLAS=cores.  Timings only (JSON)."""
    from threadpoolctl import threadpool_limits
    cores = os.cpu_count() or 1
    out = {"cores": cores}
    for name, workers, blas in (("workers=cores,BLAS=1", cores, 1), ("workers=1,BLAS=cores", 1, cores)):
        prob = ref_problem(cfg, workers=workers)
        with threadpool_limits(blas):
            t0 = time.perf_counter()
            r = rsolver.solve_direct(prob)
            wall = time.perf_counter() - t0
        out[name] = {"fill_s": r.metrics["fill_s"], "factor_s": r.metrics["factor_s"], "wall_s": wall,
                     "residual": r.residual}
        print(name, out[name], flush=True)
    path = os.path.join(HERE, f"cfg{cfg}_thread_sweep.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


def main(job):
    if job.endswith("_sweep"):
        thread_sweep(int(job[3]))
        return
    if job == "mie":
        mie_currents(2)
        mie_currents(5, n_patch=64)
        return
    cfg = int(job[3])
    what = job[5:]
    prob = ref_problem(cfg)
    if what == "class":
        gen = prob.generator()
        out = classification(gen)
        out.update({"leaf_" + k: v for k, v in sampled_leaves(prob, gen).items()})
        save(f"cfg{cfg}_class.npz", **out)
    elif what == "leaves":
        gen = prob.generator()
        lv = sampled_leaves(prob, gen, n_each=32, sub=16)
        # classification of the patch columns the sampled leaves touched
        pids = sorted({pid for (pt, pid) in gen._class_cache.keys()})[:12]
        cl = classification(prob.generator(), pids)
        out = {"leaf_" + k: v for k, v in lv.items()}
        out.update(cl)
        save(f"cfg{cfg}_class.npz", **out)
    elif what == "solve":
        save(f"cfg{cfg}_solve.npz", **solve(prob))
    elif what == "dense":
        save(f"cfg{cfg}_dense.npz", **solve(prob, dense=True))
    else:
        raise SystemExit(f"unknown job {job}")


if __name__ == "__main__":
    for j in sys.argv[1:]:
        main(j)
