import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17116_b200 import configs, hmatrix as hm
cfg = int(sys.argv[1])
prob = configs.problem(cfg)
t = time.perf_counter(); gen = prob.generator(); print("setup+classify s", time.perf_counter() - t, gen.stats(), flush=True)
t = time.perf_counter(); H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol); print("hmatrix s", time.perf_counter() - t, json.dumps(H.stats()), flush=True)
if len(sys.argv) > 2 and sys.argv[2] == "fill":
    sys.exit(0)
t = time.perf_counter(); F = hm.hlu_factor(H, prob.aca_tol); print("hlu s", time.perf_counter() - t, json.dumps(F.stats()), flush=True)
b = gen.rhs(prob.excitation) * gen.row_scale
import numpy as np
x = F.solve(b)
print("residual", np.linalg.norm(H.matvec(x) - b) / np.linalg.norm(b), flush=True)
