"""Time the public-API path of bench.py's e2e leg piece by piece (config 2)."""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from paper_2408_17116_b200 import configs, hmatrix as hm  # noqa: E402
from paper_2408_17116_b200.solver import build_hmatrix  # noqa: E402

prob = configs.problem(2)
for it in range(4):
    t0 = time.perf_counter()
    H2, gen2, scaled2, _ = build_hmatrix(dataclasses.replace(prob))
    t1 = time.perf_counter()
    F2 = hm.hlu_factor(H2, prob.effective_trunc_tol)
    t2 = time.perf_counter()
    rhs = gen2.rhs(prob.excitation) * scaled2.row_scale
    x = F2.solve(rhs) * scaled2.col_scale
    t3 = time.perf_counter()
    st = F2.stats()
    del H2, gen2, F2
    t4 = time.perf_counter()
    print(f"it {it}: build {1e3*(t1-t0):.1f} factor {1e3*(t2-t1):.1f} (dev {st['factor_device_ms']:.1f} "
          f"rec {st['record_ms']:.1f} cached {st['plan_cached']}) solve {1e3*(t3-t2):.1f} del {1e3*(t4-t3):.1f}",
          flush=True)
