"""H-LU device time (3 factorisations, warm plan) + residual of one solve, configs on argv."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

for cfg in [int(a) for a in sys.argv[1:]]:
    prob = configs.problem(cfg)
    gen = prob.generator()
    H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
    ts = []
    for it in range(3):
        F = hm.hlu_factor(H, prob.effective_trunc_tol)
        st = F.stats()
        ts.append(round(st["factor_device_ms"], 2))
        if it < 2:
            del F
    b = gen.rhs(prob.excitation) * gen.row_scale
    res = float(np.linalg.norm(H.matvec(F.solve(b)) - b) / np.linalg.norm(b))
    print(json.dumps({"cfg": cfg, "fill_ms": H.stats()["fill_ms"], "hlu_ms": ts, "residual": res,
                      "overflow": st["trunc_overflow"], "record_ms": st["record_ms"],
                      "solve_ms": F.stats().get("solve_device_ms"), "levels": st.get("levels"),
                      "launches": st.get("launches"), "temp_gb": round(st.get("temp_bytes", 0) / 2 ** 30, 1),
                      "pool_gb": round(st.get("pool_budget_gb", 0), 1),
                      "tflops": round(st.get("flops", 0) / st["factor_device_ms"] / 1e9, 2)}), flush=True)
    del F, H, gen
