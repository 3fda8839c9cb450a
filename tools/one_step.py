"""One fill + H-LU pass of a configuration (the unit ncu captures profile)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

prob = configs.problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
F = hm.hlu_factor(H, prob.effective_trunc_tol)
print("ok", F.stats()["factor_device_ms"])
