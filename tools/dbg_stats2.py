"""Factor config N twice (second run hits the plan cache) and print both stat sets."""
import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_2408_17116_b200 import configs, hmatrix as hm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
keys = sys.argv[2].split(",") if len(sys.argv) > 2 else None
prob = configs.problem(cfg)
gen = prob.generator()
for it in range(2):
    H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
    F = hm.hlu_factor(H, prob.aca_tol)
    st = F.stats()
    print(it, json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in st.items()
                          if keys is None or any(k.startswith(q) for q in keys)}))
    del H, F
