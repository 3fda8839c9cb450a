"""Fill + factor config N once with CBIE_PROFILE=1 semantics (per-kind device ms) and print the stats."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CBIE_PROFILE", "1")
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = configs.problem(cfg)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
print("hmatrix", json.dumps(H.stats()), flush=True)
F = hm.hlu_factor(H, prob.effective_trunc_tol)
print("hlu", json.dumps({k: round(v, 3) if isinstance(v, float) else v for k, v in F.stats().items()}), flush=True)
