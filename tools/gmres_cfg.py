"""Device GMRES on config N (default 2): iterations, residual, time, agreement with H-LU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2408_17116_b200 import configs  # noqa: E402
from paper_2408_17116_b200.solver import solve_direct, solve_gmres  # noqa: E402

prob = configs.problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
t0 = time.perf_counter()
rg = solve_gmres(prob)
t1 = time.perf_counter()
rd = solve_direct(prob)
print(f"gmres: iters {rg.iterations} converged {rg.converged} rel {rg.residual:.3e} solve_s {rg.metrics['solve_s']:.3f} "
      f"wall {t1 - t0:.2f}; direct residual {rd.residual:.3e}; "
      f"|x_g - x_d|/|x_d| {np.linalg.norm(rg.solution - rd.solution) / np.linalg.norm(rd.solution):.3e}", flush=True)
