"""Critical path of the H-LU schedule (CBIE_PROFILE + CBIE_CRIT_DUMP) for config argv[1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CBIE_PROFILE"] = "1"
os.environ["CBIE_CRIT_DUMP"] = "1"
os.environ.setdefault("CBIE_TRUNC_DUMP", "1")
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prob = configs.problem(cfg)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
F = hm.hlu_factor(H, prob.effective_trunc_tol)
print({k: v for k, v in F.stats().items() if k.startswith(("crit", "factor", "trunc_n", "trunc_cyc"))})
