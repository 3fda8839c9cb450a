import os, sys
sys.path.insert(0, os.getcwd())
from paper_2408_17116_b200 import configs, hmatrix as hm
prob = configs.problem(1)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
F = hm.hlu_factor(H, prob.aca_tol)
print("ok", F.stats()["levels"])
