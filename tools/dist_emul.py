"""Distributed H-LU plan emulated on one GPU for config N with W virtual ranks:
factor single + emulated, compare solutions, print the plan statistics."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2408_17116_b200 import configs, hmatrix as hm

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
worlds = [int(w) for w in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "4"])]
prob = configs.problem(cfg)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
b = gen.rhs(prob.excitation)
F1 = hm.hlu_factor(H, prob.effective_trunc_tol)
x1 = F1.solve(b)
res1 = float(np.linalg.norm(H.matvec(x1) - b) / np.linalg.norm(b))
del F1
for W in worlds:
    t0 = time.perf_counter()
    Fd = hm.hlu_factor(H, prob.effective_trunc_tol, emulate_world=W)
    t1 = time.perf_counter()
    xd = Fd.solve(b)
    st = {k: v for k, v in Fd.stats().items() if k.startswith("dist_") or k in ("factor_device_ms", "record_ms")}
    out = {"cfg": cfg, "world": W, "wall_s": t1 - t0, "rel_vs_single": float(np.linalg.norm(xd - x1) / np.linalg.norm(x1)),
           "residual_single": res1, "residual_dist": float(np.linalg.norm(H.matvec(xd) - b) / np.linalg.norm(b)), **st}
    print(json.dumps(out), flush=True)
    del Fd
