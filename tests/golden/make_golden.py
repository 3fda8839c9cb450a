"""Generate golden fixtures by running the REFERENCE package (read-only).

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every array written here comes from the reference's own public functions; the
oracle (oracle/) and the CUDA path are pinned against these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from chebscat import assembly as asm           # noqa: E402
from chebscat import chebyshev as cheb         # noqa: E402
from chebscat import geometry as geo           # noqa: E402
from chebscat import hmatrix as hm             # noqa: E402
from chebscat import kernels as ker            # noqa: E402
from chebscat import postprocess as post       # noqa: E402
from chebscat import quadrature as quad        # noqa: E402
from chebscat.solver import Problem, solve_dense, solve_direct  # noqa: E402

THETA = np.linspace(0.0, 180.0, 181)


def save(name, **arrs):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)")


def spectral():
    out = {}
    rng = np.random.default_rng(11)
    for n in (4, 5, 6, 8, 16):
        r = cheb.fejer1(n)
        out[f"fejer_x_{n}"] = r.nodes
        out[f"fejer_w_{n}"] = r.weights
        out[f"dnode_{n}"] = cheb.diff_node_matrix(n)
    u = rng.uniform(-1, 1, 40)
    v = rng.uniform(-1, 1, 40)
    P, dU, dV = cheb.cardinal_eval((6, 8), u, v)
    out.update(card_u=u, card_v=v, card_P=P, card_dU=dU, card_dV=dV)
    c = rng.standard_normal((6, 8))
    out.update(clen_c=c, clen_val=cheb.eval2d_raw(c, u, v))
    save("spectral.npz", **out)


def mfie_problem(radius, refinement, order, **kw):
    med = ker.Medium.from_relative(1.0, 1.0, 1.0)
    spec = ker.FormulationSpec(ker.MFIE_PEC, med)
    pw = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
    return Problem(geo.unit_sphere_patches(radius, refinement, order), spec, pw, **kw)


def muller_problem(radius, refinement, order, eps2, **kw):
    med1 = ker.Medium.from_relative(1.0, 1.0, 1.0)
    med2 = ker.Medium.from_relative(eps2, 1.0, 1.0)
    spec = ker.FormulationSpec(ker.MULLER, med1, med2)
    pw = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
    return Problem(geo.unit_sphere_patches(radius, refinement, order), spec, pw, **kw)


def geometry(prob):
    rng = np.random.default_rng(12)
    p = prob.patches[5]
    u = rng.uniform(-1, 1, 30)
    v = rng.uniform(-1, 1, 30)
    fb = geo.eval_frames(p, u, v)
    ruu, ruv, rvv = geo.second_derivatives(p, u, v)
    # same patch without its chart: Chebyshev-interpolated geometry
    q = geo.Patch(99, p.samples.copy())
    fq = geo.eval_frames(q, u, v)
    save("geometry.npz", samples=p.samples, u=u, v=v, pos=fb.position, au=fb.a_u,
         av=fb.a_v, sg=fb.sqrt_g, ruu=ruu, ruv=ruv, rvv=rvv,
         cheb_pos=fq.position, cheb_au=fq.a_u, cheb_av=fq.a_v, cheb_sg=fq.sqrt_g,
         diam=p.diameter)


def classification(prob, name):
    gen = prob.generator()
    P = len(prob.patches)
    rec = []
    for pid in range(P):
        gen._classify_patch_column(pid)
    for (pt, pid), ic in gen._class_cache.items():
        if ic.tag == quad.FAR:
            continue
        rec.append((pt, pid, 1 if ic.tag == quad.NEAR else 2, ic.uv[0], ic.uv[1],
                    1 if ic.newton_ok else 0))
    rec.sort()
    a = np.array(rec, dtype=float)
    save(name, point=a[:, 0].astype(np.int32), patch=a[:, 1].astype(np.int32),
         tag=a[:, 2].astype(np.int8), u=a[:, 3], v=a[:, 4], ok=a[:, 5].astype(np.int8),
         fallbacks=gen.newton_fallbacks, npts=gen.dofmap.n_points, npatch=P)
    return gen


def pair_blocks(gen, name, n_each=12, seed=13):
    rng = np.random.default_rng(seed)
    by = {quad.SELF: [], quad.NEAR: [], quad.FAR: []}
    for key, ic in gen._class_cache.items():
        by[ic.tag].append(key)
    keys = []
    for tag in (quad.SELF, quad.NEAR, quad.FAR):
        lst = sorted(by[tag])
        idx = rng.choice(len(lst), size=min(n_each, len(lst)), replace=False)
        keys += [lst[i] for i in sorted(idx)]
    blocks = np.stack([gen.pair_block(p, q) for p, q in keys])
    save(name, keys=np.array(keys, dtype=np.int32), blocks=blocks)


def dense_entries(gen, name, n=3000, seed=14):
    rng = np.random.default_rng(seed)
    N = gen.dofmap.n_dofs
    ii = rng.integers(0, N, n)
    jj = rng.integers(0, N, n)
    vals = np.array([gen.entry(int(i), int(j)) for i, j in zip(ii, jj)])
    save(name, i=ii, j=jj, val=vals)


def tree_and_solve(prob, name, dense=True):
    rd = solve_direct(prob)
    gen = prob.generator()
    pts = gen.dofmap.point_positions()
    tree = hm.build_cluster_tree(pts, prob.spec.n_components, prob.n_leaf)
    H = hm.build_block_tree(tree, prob.eta)
    leaves = []

    def walk(b, r, c):
        if isinstance(b, hm.HBlock):
            for a, rk in enumerate(b.rows):
                for k, ck in enumerate(b.cols):
                    walk(b.children[a][k], rk, ck)
        else:
            leaves.append((r.lo, r.hi, c.lo, c.hi, 1 if isinstance(b, hm._PendingLowRank) else 0))

    walk(H.root, tree.root, tree.root)
    out = dict(dof_perm=tree.dof_perm, leaves=np.array(leaves, dtype=np.int64),
               x_direct=rd.solution, residual=rd.residual,
               compression=rd.metrics["compression_rate"],
               demoted=rd.metrics["hmatrix_diagnostics"]["demoted_blocks"],
               fallbacks=rd.metrics["newton_fallbacks"])
    cut = post.rcs_cut(prob, rd.solution, 0.0, THETA)
    out["rcs_direct_db"] = cut.sigma_dbsm
    if dense:
        rf = solve_dense(prob)
        out["x_dense"] = rf.solution
        out["rcs_dense_db"] = post.rcs_cut(prob, rf.solution, 0.0, THETA).sigma_dbsm
    rhs = asm.rhs(prob.patches, prob.spec, prob.excitation)
    out["rhs"] = rhs
    save(name, **out)


def aca_kat():
    rng = np.random.default_rng(15)
    n1, n2 = 60, 50
    a1 = rng.standard_normal((n1, 3))
    a1 /= np.linalg.norm(a1, axis=1, keepdims=True)
    a2 = rng.standard_normal((n2, 3))
    a2 /= np.linalg.norm(a2, axis=1, keepdims=True)
    p1 = 0.4 * a1
    p2 = 0.4 * a2 + np.array([4.0, 0.0, 0.0])
    R = np.linalg.norm(p1[:, None] - p2[None, :], axis=-1)
    M = np.exp(-1j * 2 * np.pi * R) / (4 * np.pi * R)
    U, V = hm.aca(lambda i: M[i].copy(), lambda j: M[:, j].copy(), n1, n2, 1e-4)
    Ut, Vt = hm.truncate_lowrank(np.concatenate([U, 0.3 * U[:, :2]], 1),
                                 np.concatenate([V, V[:2] * 1j], 0), 1e-6)
    save("aca.npz", M=M, UV=U @ V, rank=U.shape[1], trunc_UV=Ut @ Vt, trunc_rank=Ut.shape[1])


if __name__ == "__main__":
    which = sys.argv[1:] or ["spectral", "cfg1", "small", "muller", "aca"]
    if "spectral" in which:
        spectral()
    if "aca" in which:
        aca_kat()
    if "cfg1" in which:
        prob = mfie_problem(0.5, 1, (6, 6), aca_tol=1e-6, eta=1.0, n_leaf=128)
        geometry(prob)
        gen = classification(prob, "cfg1_class.npz")
        pair_blocks(gen, "cfg1_pairs.npz")
        dense_entries(gen, "cfg1_entries.npz")
        tree_and_solve(prob, "cfg1_solve.npz")
    if "small" in which:
        prob = mfie_problem(0.5, 0, (4, 4))
        tree_and_solve(prob, "small_solve.npz")
    if "muller" in which:
        prob = muller_problem(0.5, 0, (5, 5), 4.0, aca_tol=1e-5)
        gen = classification(prob, "muller_class.npz")
        pair_blocks(gen, "muller_pairs.npz", n_each=8)
        tree_and_solve(prob, "muller_solve.npz")
