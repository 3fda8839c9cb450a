"""Solve-phase statistics of config 2 (levels, launches per kind, device time)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

prob = configs.problem(2)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
F = hm.hlu_factor(H, prob.effective_trunc_tol)
b = gen.rhs(prob.excitation)
for it in range(4):
    t0 = time.perf_counter()
    F.solve(b)
    t1 = time.perf_counter()
    print(f"solve {1e3 * (t1 - t0):.1f} ms", json.dumps(F.solve_stats()), flush=True)
