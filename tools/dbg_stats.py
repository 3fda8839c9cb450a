import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_2408_17116_b200 import configs, hmatrix as hm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = configs.problem(cfg)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
F = hm.hlu_factor(H, prob.aca_tol)
print(json.dumps({k: v for k, v in F.stats().items()}, indent=0))
