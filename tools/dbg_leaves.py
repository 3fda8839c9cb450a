import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2408_17116_b200 import configs, hmatrix as hm
from oracle import pipeline as pl
prob = configs.problem(1)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
A = pl.case(1).disc().dense()
perm, lv = H.tree()
C = 2
bad = []
for i, row in enumerate(lv):
    rows = perm[row[0] * C:row[1] * C]; cols = perm[row[2] * C:row[3] * C]
    ref = A[np.ix_(rows, cols)]
    lf = H.leaf(i)
    M = lf[1] if lf[0] == "dense" else lf[1] @ lf[2]
    e = np.linalg.norm(M - ref) / np.linalg.norm(ref)
    bad.append((e, i, lf[0], int(row[5]), tuple(row[:4])))
bad.sort(reverse=True)
for b in bad[:12]: print(b)
print(H.stats())
