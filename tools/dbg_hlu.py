import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2408_17116_b200 import geometry as geo, kernels as ker
from paper_2408_17116_b200.solver import Problem, solve_direct
vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
pw = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
for (rad, ref, order, leaf, tol) in [(1.0, 2, 4, 64, 1e-4), (1.0, 2, 4, 128, 1e-4), (2.0, 2, 6, 256, 1e-4), (2.0, 2, 8, 256, 1e-4)]:
    prob = Problem(geo.unit_sphere_patches(rad, ref, (order, order)), ker.FormulationSpec(ker.MFIE_PEC, vac), pw, aca_tol=tol, eta=1.0, n_leaf=leaf)
    t = time.perf_counter(); r = solve_direct(prob); t = time.perf_counter() - t
    h = r.metrics["device"]["hlu"]
    print(rad, ref, order, leaf, "N", prob.n_dofs, "res", r.residual, "t", round(t, 2), {k: (round(v, 1) if isinstance(v, float) else v) for k, v in h.items() if k.startswith(("ms_", "tasks_", "launch_", "levels", "temp"))}, flush=True)
