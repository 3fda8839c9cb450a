"""End-to-end pipelines (drop-in for chebscat.solver: Problem, build_hmatrix,
solve_direct, solve_dense; solver.py:30-203).  Same Problem fields and the
same SolveResult metric keys, plus device timings from CUDA events."""

from __future__ import annotations

import resource
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import assembly as asm
from . import hmatrix as hm
from .kernels import FormulationSpec, PlaneWave


@dataclass
class Problem:
    patches: list
    spec: FormulationSpec
    excitation: PlaneWave
    aca_tol: float = 1e-4
    trunc_tol: Optional[float] = None
    gmres_tol: float = 1e-4
    gmres_restart: int = 200
    gmres_max_iters: int = 2000
    eta: float = 2.0
    n_leaf: int = 64
    tau: float = 1.0
    grading: int = 3
    oversample: Optional[int] = None
    dense_cap: int = asm.DENSE_CAP_DEFAULT
    workers: int = 1          # no meaning on the GPU path
    device: int = 0

    def __post_init__(self):
        for name in ("aca_tol", "gmres_tol"):
            v = getattr(self, name)
            if not (0.0 < v < 1.0):
                raise ValueError(f"{name} must lie in (0, 1), got {v}")
        if self.trunc_tol is not None and not (0.0 < self.trunc_tol < 1.0):
            raise ValueError("trunc_tol must lie in (0, 1)")

    @property
    def effective_trunc_tol(self) -> float:
        return self.aca_tol if self.trunc_tol is None else self.trunc_tol

    def generator(self) -> asm.GpuGenerator:
        return asm.GpuGenerator(self.patches, self.spec, tau=self.tau,
                                oversample=self.oversample, grading=self.grading,
                                device=self.device)

    @property
    def n_dofs(self) -> int:
        return sum(p.n_nodes for p in self.patches) * self.spec.n_components


@dataclass
class SolveResult:
    solution: np.ndarray
    residual: float
    metrics: dict = field(default_factory=dict)
    iterations: int = 0
    converged: bool = True


def _chart_from_reference(ch):
    """Device chart for a reference ``Chart`` (geometry.py:38-97)."""
    from . import geometry as geo
    if ch is None or isinstance(ch, (geo.CubeSphereFace,)):
        return ch
    box = tuple(getattr(ch, a, None) for a in ("radius", "face", "u_lo", "u_hi", "v_lo", "v_hi"))
    if None in box:
        raise ValueError(f"chart {type(ch).__name__} has no device evaluator "
                         "(supported: CubeSphereFace, the config-4 star chart, chart-less patches)")
    if getattr(ch, "coef", None) is not None:               # star chart (config 4)
        return geo.StarFace(*box, coef=np.asarray(ch.coef, float))
    if type(ch).__name__ == "CubeSphereFace":
        return geo.CubeSphereFace(*box)
    raise ValueError(f"chart {type(ch).__name__} has no device evaluator")


def from_reference(problem) -> "Problem":
    """This package's Problem for a reference ``chebscat.solver.Problem`` (solver.py:30-73)
    built from chebscat's own Patch / CubeSphereFace / FormulationSpec / Medium /
    PlaneWave / Dipole objects.  Samples, chart parameters, media and solver settings
    are taken over unchanged; a Problem of this package is returned as is."""
    from . import geometry as geo
    from . import kernels as ker
    if isinstance(problem, Problem):
        return problem
    patches = [geo.Patch(int(p.id), np.array(p.samples, float), chart=_chart_from_reference(p.chart))
               for p in problem.patches]

    def med(m):
        return None if m is None else ker.Medium(complex(m.eps), complex(m.mu), float(m.omega))

    spec = ker.FormulationSpec(str(problem.spec.kind), med(problem.spec.outer), med(problem.spec.inner))
    exc = problem.excitation
    if hasattr(exc, "polarization"):
        exc = ker.PlaneWave(np.array(exc.direction, float), np.array(exc.polarization, float),
                            float(exc.amplitude))
    else:
        exc = ker.Dipole(np.array(exc.position, float), np.array(exc.moment, float))
    keys = ("aca_tol", "trunc_tol", "gmres_tol", "gmres_restart", "gmres_max_iters", "eta", "n_leaf",
            "tau", "grading", "oversample", "dense_cap", "workers")
    kw = {k: getattr(problem, k) for k in keys if hasattr(problem, k)}
    return Problem(patches, spec, exc, **kw)


def _peak_rss_bytes() -> int:
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024


def build_hmatrix(problem: Problem, gen: Optional[asm.GpuGenerator] = None):
    """Classification + near field + H-matrix fill of the scaled system."""
    problem = from_reference(problem)
    t0 = time.perf_counter()
    gen = gen or problem.generator()
    t1 = time.perf_counter()
    H = hm.HMatrix(gen, problem.n_leaf, problem.eta, problem.aca_tol)
    t2 = time.perf_counter()
    st = H.stats()
    gs = gen.stats()
    times = {"setup_s": t1 - t0, "fill_s": t2 - t1, "tree_s": st.get("tree_ms", 0) / 1e3,
             "device_fill_s": (gs.get("classify_ms", 0) + gs.get("near_fill_ms", 0)
                               + st.get("fill_ms", 0)) / 1e3}
    return H, gen, asm.ScaledView(gen), times


def solve_direct(problem: Problem) -> SolveResult:
    """H-matrix fill, H-LU, forward/backward substitution (solver.py:148-175)."""
    problem = from_reference(problem)
    H, gen, scaled, times = build_hmatrix(problem)
    b = gen.rhs(problem.excitation)
    b_scaled = b * scaled.row_scale
    t0 = time.perf_counter()
    F = hm.hlu_factor(H, problem.effective_trunc_tol)
    t_factor = time.perf_counter() - t0
    t0 = time.perf_counter()
    x = F.solve(b_scaled) * scaled.col_scale
    t_solve = time.perf_counter() - t0
    bnorm = np.linalg.norm(b_scaled)
    residual = float(np.linalg.norm(H.matvec(x / scaled.col_scale) - b_scaled) / bnorm) \
        if bnorm else 0.0
    metrics = {
        **times,
        "factor_s": t_factor,
        "solve_s": t_solve,
        "n_dofs": problem.n_dofs,
        "hmatrix_bytes": H.memory_bytes(),
        "hlu_bytes": F.memory_bytes(),
        "compression_rate": H.compression_rate(),
        "peak_rss_bytes": _peak_rss_bytes(),
        "memory_method": "ru_maxrss sampling + logical leaf accounting",
        "hmatrix_diagnostics": H.diagnostics(),
        "newton_fallbacks": gen.newton_fallbacks,
        "device": {"generator": gen.stats(), "hmatrix": H.stats(), "hlu": F.stats()},
    }
    return SolveResult(x, residual, metrics)


def solve_gmres(problem: Problem, restart: Optional[int] = None,
                max_iters: Optional[int] = None) -> SolveResult:
    """Unpreconditioned restarted GMRES on the compressed operator (solver.py:206-307):
    the Krylov basis, the H-matvec and every vector operation stay on the device
    (cbie_gmres, csrc/gmres.cu)."""
    import ctypes as ct
    from . import _ffi
    problem = from_reference(problem)
    restart = restart if restart is not None else problem.gmres_restart
    max_iters = max_iters if max_iters is not None else problem.gmres_max_iters
    dense = problem.n_dofs <= 600
    if dense:
        # the reference iterates on the dense equilibrated matrix up to N = 600
        # (solver.py:278-287): one dense leaf covering the whole matrix -- the device
        # matvec is then the exact dense product of the same scaled entries
        import dataclasses
        H, gen, scaled, times = build_hmatrix(dataclasses.replace(problem, n_leaf=max(problem.n_leaf,
                                                                                       problem.n_dofs)))
    else:
        H, gen, scaled, times = build_hmatrix(problem)
    b = np.ascontiguousarray(gen.rhs(problem.excitation) * scaled.row_scale)
    y = np.empty_like(b)
    it, rel, ok = ct.c_int(), ct.c_double(), ct.c_int()
    t0 = time.perf_counter()
    H.dev.check(H.dev.lib.cbie_gmres(H.h, _ffi.ptr(b), float(problem.gmres_tol), int(restart), int(max_iters),
                                     _ffi.ptr(y), ct.byref(it), ct.byref(rel), ct.byref(ok)))
    t_solve = time.perf_counter() - t0
    x = y * scaled.col_scale
    metrics = {**times, "operator": "dense" if dense else "hmatrix", "solve_s": t_solve,
               "n_dofs": problem.n_dofs, "hmatrix_bytes": H.memory_bytes(),
               "compression_rate": H.compression_rate(), "peak_rss_bytes": _peak_rss_bytes(),
               "memory_method": "ru_maxrss sampling + logical leaf accounting"}
    return SolveResult(x, float(rel.value), metrics, iterations=int(it.value), converged=bool(ok.value))


def solve_dense(problem: Problem) -> SolveResult:
    """Dense fill + LU with partial pivoting + solve of the unscaled system, all on the
    device (solver.py:178-203; cbie_dense_solve, csrc/dense_solve.cu)."""
    import ctypes as ct
    from . import _ffi
    problem = from_reference(problem)
    gen = problem.generator()
    b = np.ascontiguousarray(gen.rhs(problem.excitation).reshape(-1, 1))
    x = np.empty_like(b)
    res = ct.c_double()
    t0 = time.perf_counter()
    gen.dev.check(gen.dev.lib.cbie_dense_solve(gen.dev.h, int(problem.dense_cap), _ffi.ptr(b), 1, _ffi.ptr(x),
                                               ct.byref(res), None, None))
    wall = time.perf_counter() - t0
    st = gen.stats()
    return SolveResult(x[:, 0], float(res.value),
                       {"fill_s": st.get("dense_fill_ms", 0.0) / 1e3, "factor_s": st.get("dense_lu_ms", 0.0) / 1e3,
                        "solve_s": st.get("dense_solve_ms", 0.0) / 1e3, "wall_s": wall,
                        "n_dofs": problem.n_dofs, "dense_bytes": 16 * problem.n_dofs ** 2,
                        "peak_rss_bytes": _peak_rss_bytes(),
                        "memory_method": "ru_maxrss sampling + logical array accounting",
                        "newton_fallbacks": gen.newton_fallbacks})
