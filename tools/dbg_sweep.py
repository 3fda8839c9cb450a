import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2408_17116_b200 import geometry as geo, kernels as ker
from paper_2408_17116_b200.solver import Problem, solve_direct
vac = ker.Medium.from_relative(1.0, 1.0, 1.0)
pw = ker.PlaneWave([0, 0, 1], [1, 0, 0], 1.0)
cases = [tuple(map(float, c.split(","))) for c in sys.argv[1:]]
for (rad, ref, order, leaf, tol) in cases:
    prob = Problem(geo.unit_sphere_patches(rad, int(ref), (int(order), int(order))), ker.FormulationSpec(ker.MFIE_PEC, vac), pw, aca_tol=tol, eta=1.0, n_leaf=int(leaf))
    t = time.perf_counter(); r = solve_direct(prob); t = time.perf_counter() - t
    h = r.metrics["device"]["hlu"]
    print(rad, ref, order, leaf, tol, "N", prob.n_dofs, "res %.3e" % r.residual, "t %.1f" % t, "levels", h["levels"], "ovf", h["trunc_overflow"], "CR %.3f" % r.metrics["compression_rate"], flush=True)
