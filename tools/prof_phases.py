"""Gram-path phase breakdown (mean cycles per problem) for config argv[1]; CBIE_PROF_MN /
CBIE_PROF_KMIN restrict the mean to large blocks / large concatenated ranks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CBIE_PROFILE", "1")
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prob = configs.problem(cfg)
gen = prob.generator()
H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
F = hm.hlu_factor(H, prob.effective_trunc_tol)
st = F.stats()
print(json.dumps({"mn": os.environ.get("CBIE_PROF_MN"), "kmin": os.environ.get("CBIE_PROF_KMIN"),
                  **{k: round(v, 1) for k, v in st.items() if k.startswith(("gram_cyc", "trunc_cyc", "trunc_mean"))}}))
