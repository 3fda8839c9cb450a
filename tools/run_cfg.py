"""Run one configuration end to end on the GPU and print timings / parity numbers."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from paper_2408_17116_b200 import configs
from paper_2408_17116_b200.solver import solve_direct

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = configs.problem(cfg)
t0 = time.perf_counter()
r = solve_direct(prob)
t1 = time.perf_counter()
m = r.metrics
out = {"cfg": cfg, "N": prob.n_dofs, "wall_s": t1 - t0, "residual": r.residual,
       "fill_s": m["fill_s"], "factor_s": m["factor_s"], "solve_s": m["solve_s"],
       "compression": m["compression_rate"], "gen": m["device"]["generator"],
       "hmat": m["device"]["hmatrix"], "hlu": m["device"]["hlu"]}
if cfg == 1:
    from gold import golden
    g = golden("cfg1_solve.npz")
    out["rel_vs_ref_direct"] = float(np.linalg.norm(r.solution - g["x_direct"]) / np.linalg.norm(g["x_direct"]))
    out["rel_vs_ref_dense"] = float(np.linalg.norm(r.solution - g["x_dense"]) / np.linalg.norm(g["x_dense"]))
print(json.dumps(out, indent=1))
