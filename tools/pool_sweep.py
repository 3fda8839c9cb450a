"""H-LU device time vs the temporary-pool budget (CBIE_POOL_GB), config given on argv."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = configs.problem(cfg)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
for gb in sys.argv[2:]:
    if gb == "default":
        os.environ.pop("CBIE_POOL_GB", None)
    else:
        os.environ["CBIE_POOL_GB"] = gb
    out = []
    for it in range(3):
        F = hm.hlu_factor(H, prob.effective_trunc_tol)
        st = F.stats()
        out.append({k: round(st[k], 2) for k in ("factor_device_ms", "record_ms", "host_enqueue_ms",
                                                  "temp_bytes", "levels", "launches", "trunc_overflow",
                                                  "plan_cached")})
        del F
    print(json.dumps({"cfg": cfg, "pool_gb": gb, "runs": out}), flush=True)
