"""Factor the GPU H-matrix with the oracle H-LU (CPU) and with the GPU, compare leaves."""
import os, sys, time, copy
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2408_17116_b200 import geometry as geo, kernels as ker, hmatrix as hm
from paper_2408_17116_b200.solver import Problem, build_hmatrix
from oracle import hcompress as hc, hfactor as hf
rad, ref, order, leaf, tol = [float(x) for x in sys.argv[1].split(",")]
vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
pw = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
prob = Problem(geo.unit_sphere_patches(rad, int(ref), (int(order), int(order))), ker.FormulationSpec(ker.MFIE_PEC, vac), pw, aca_tol=tol, eta=1.0, n_leaf=int(leaf))
H, gen, sc, _ = build_hmatrix(prob)
Ho = hc.HMat(gen.pos, 2, int(leaf), 1.0)
lv = hc.leaves(Ho.root)
for i, b in enumerate(lv):
    l = H.leaf(i)
    if l[0] == "dense":
        b.kind = "D"; b.D = l[1]
    else:
        b.kind = "R"; b.U, b.V = l[1], l[2]
t = time.time(); Fo = hf.Factors(Ho, tol); print("oracle factor s", time.time() - t, flush=True)
F = hm.hlu_factor(H, tol)
rng = np.random.default_rng(0)
x = rng.standard_normal(H.N) + 1j * rng.standard_normal(H.N)
b = H.matvec(x)
print("oracle solve err", np.linalg.norm(Fo.solve(b) - x) / np.linalg.norm(x))
print("gpu solve err", np.linalg.norm(F.solve(b) - x) / np.linalg.norm(x), flush=True)
flv = hc.leaves(Fo.root)
bad = []
for i, ob in enumerate(flv):
    g = F.leaf(i)
    if ob.kind == "LU":
        ref_ = ob.D; got = g[1]
    elif ob.kind == "D":
        ref_ = ob.D; got = g[1]
    else:
        ref_ = ob.U @ ob.V; got = g[1] @ g[2]
    e = np.linalg.norm(got - ref_) / max(np.linalg.norm(ref_), 1e-300)
    bad.append((e, i, ob.kind, ob.r.lo, ob.r.hi, ob.c.lo, ob.c.hi, ref_.shape))
bad.sort(reverse=True)
for row in bad[:15]:
    print(row)
print("n leaves", len(flv), "n>1e-3", sum(1 for b_ in bad if b_[0] > 1e-3))
print("--- by position (first bad in factor order) ---")
bad2 = sorted(bad, key=lambda t: (min(t[3], t[5]), t[3], t[5]))
cnt = 0
for row in bad2:
    if row[0] > 1e-6:
        print(row); cnt += 1
        if cnt > 25: break
print("--- diag ---")
for row in sorted(bad, key=lambda t: t[3]):
    if row[2] == "LU":
        print(row[:3], row[3])
