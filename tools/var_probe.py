"""Repeat fill + H-LU of config 2 in one process; print device / host-enqueue times per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402

prob = configs.problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
gen = prob.generator()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    t0 = time.perf_counter()
    gen.classify()
    tc = time.perf_counter()
    H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
    t1 = time.perf_counter()
    F = hm.hlu_factor(H, prob.effective_trunc_tol)
    t2 = time.perf_counter()
    st = F.stats()
    t3 = time.perf_counter()
    del H, F
    t4 = time.perf_counter()
    print(f"step {it}: classify {1e3*(tc-t0):.1f} del {1e3*(t4-t3):.1f} fill_wall {1e3*(t1-t0):.1f} hlu_wall {1e3*(t2-t1):.1f} device {st['factor_device_ms']:.1f} "
          f"enqueue {st.get('host_enqueue_ms', 0):.1f} frees {st.get('frees_during_run', 0):.0f} "
          f"cached {st.get('plan_cached')} trunc_ms {st.get('trunc_kernel_ms', 0):.1f}", flush=True)
