"""GPU entry generator: drop-in for chebscat.assembly.EntryGenerator
(assembly.py:68-334), assemble_dense (438-460) and rhs (463-466).

The generator protocol the reference's H-matrix engine consumes
(row_segment / col_segment / block / entry, hmatrix.py:243-264) is served by
libcbie.so: classification, near pair blocks and every entry are computed on
the GPU; this class only owns the device context and marshals index arrays.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _ffi
from . import geometry as geo
from . import kernels as ker

DENSE_CAP_DEFAULT = 20_000


class Device:
    """Owns one cbie_ctx (one CUDA device)."""

    def __init__(self, device: int = 0):
        self.lib = _ffi.load()
        h = ct.c_void_p()
        rc = self.lib.cbie_create(int(device), ct.byref(h))
        if rc != 0:
            from .errors import NativeUnavailable
            raise NativeUnavailable(f"cbie_create failed (code {rc}): no usable CUDA device")
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.cbie_destroy(h)
            self.h = None

    def check(self, rc):
        _ffi.check(rc, self.h)


class GpuGenerator:
    """Deterministic on-device generator of system-matrix entries."""

    def __init__(self, patches, spec: ker.FormulationSpec, tau: float = 1.0,
                 oversample=None, grading: int = 3, device: int = 0, scaled_default=False):
        self.patches = patches
        self.spec = spec
        self.C = spec.n_components
        self.dev = Device(device)
        lib, h = self.dev.lib, self.dev.h
        smp, kind, par, star, coef = geo.device_arrays(patches)
        nu, nv = patches[0].orders
        self.nu, self.nv = nu, nv
        self.n_points = len(patches) * nu * nv
        self.n_dofs = self.n_points * self.C
        self.dev.check(lib.cbie_set_geometry(h, len(patches), nu, nv, _ffi.ptr(smp),
                                             _ffi.ptr(kind), _ffi.ptr(par),
                                             _ffi.ptr(star) if star is not None else None,
                                             _ffi.ptr(coef)))
        outer = spec.outer
        inner = spec.inner or outer
        rsc, csc = spec.scales()
        self.row_c, self.col_c = rsc, csc
        rsc = np.ascontiguousarray(rsc, complex)
        csc = np.ascontiguousarray(csc, complex)
        kind_id = 0 if spec.kind == ker.MFIE_PEC else 1
        self.dev.check(lib.cbie_set_formulation(
            h, kind_id, float(outer.omega), _ffi.c128(outer.k), _ffi.c128(inner.k),
            _ffi.c128(outer.eps), _ffi.c128(outer.mu), _ffi.c128(inner.eps), _ffi.c128(inner.mu),
            float(tau), int(grading), int(oversample or 0), _ffi.ptr(rsc), _ffi.ptr(csc)))
        nn, ns, nf = ct.c_int64(), ct.c_int64(), ct.c_int64()
        self.dev.check(lib.cbie_classify(h, ct.byref(nn), ct.byref(ns), ct.byref(nf)))
        self.n_near, self.n_self, self.newton_fallbacks = nn.value, ns.value, nf.value
        n = self.n_points
        self.pos = np.empty((n, 3))
        self.a_u = np.empty((n, 3))
        self.a_v = np.empty((n, 3))
        self.sqrt_g = np.empty(n)
        self.dev.check(lib.cbie_node_frames(h, _ffi.ptr(self.pos), _ffi.ptr(self.a_u),
                                            _ffi.ptr(self.a_v), _ffi.ptr(self.sqrt_g)))
        self.row_scale = np.tile(self.row_c, n)
        self.col_scale = np.tile(self.col_c, n)

    def classify(self):
        """Re-run classification + near-field pair blocks on the device (one
        pass of the fill's K1/K3 stage; the geometry stays resident)."""
        nn, ns, nf = ct.c_int64(), ct.c_int64(), ct.c_int64()
        self.dev.check(self.dev.lib.cbie_classify(self.dev.h, ct.byref(nn), ct.byref(ns), ct.byref(nf)))
        self.n_near, self.n_self, self.newton_fallbacks = nn.value, ns.value, nf.value

    @property
    def stream(self) -> int:
        return int(self.dev.lib.cbie_stream(self.dev.h) or 0)

    # -- classification export -------------------------------------------------------
    def classification(self):
        m = self.n_near + self.n_self
        out = dict(point=np.empty(m, np.int32), patch=np.empty(m, np.int32),
                   tag=np.empty(m, np.int8), u=np.empty(m), v=np.empty(m), ok=np.empty(m, np.int8))
        self.dev.check(self.dev.lib.cbie_export_classification(
            self.dev.h, m, *(_ffi.ptr(out[k]) for k in ("point", "patch", "tag", "u", "v", "ok"))))
        return out

    def point_positions(self):
        return self.pos

    # -- generator protocol ---------------------------------------------------------------
    def pair_block(self, point_id: int, pid: int) -> np.ndarray:
        out = np.empty((self.C, self.nu * self.nv * self.C), complex)
        self.dev.check(self.dev.lib.cbie_pair_block(self.dev.h, int(point_id), int(pid), _ffi.ptr(out)))
        return out

    def block(self, rows, cols, fast: bool = True, scaled: bool = False) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty((rows.size, cols.size), complex)
        self.dev.check(self.dev.lib.cbie_fill_block(self.dev.h, _ffi.ptr(rows), rows.size,
                                                    _ffi.ptr(cols), cols.size, int(scaled),
                                                    _ffi.ptr(out)))
        return out

    def entry(self, i: int, j: int) -> complex:
        return complex(self.block([i], [j])[0, 0])

    def row_segment(self, i: int, cols) -> np.ndarray:
        return self.block([i], cols)[0]

    def col_segment(self, rows, j: int) -> np.ndarray:
        return self.block(rows, [j])[:, 0]

    def rhs(self, exc: ker.PlaneWave) -> np.ndarray:
        return ker.rhs_rows(self.spec, exc, self.pos, self.a_u, self.a_v).reshape(-1)

    def stats(self) -> dict:
        return _ffi.stats(self.dev.h, 0)


class ScaledView:
    """EquilibratedGenerator (solver.py:90-129) over a GpuGenerator, scaling on device."""

    def __init__(self, gen: GpuGenerator):
        self.base = gen
        self.row_scale = gen.row_scale
        self.col_scale = gen.col_scale

    def row_segment(self, i, cols):
        return self.base.block([i], cols, scaled=True)[0]

    def col_segment(self, rows, j):
        return self.base.block(rows, [j], scaled=True)[:, 0]

    def block(self, rows, cols, fast: bool = True):
        return self.base.block(rows, cols, scaled=True)


def assemble_dense(gen: GpuGenerator, cap: int = DENSE_CAP_DEFAULT, workers: int = 1) -> np.ndarray:
    """Full (unscaled) matrix on the GPU; CapExceeded if N > cap."""
    A = np.empty((gen.n_dofs, gen.n_dofs), complex)
    gen.dev.check(gen.dev.lib.cbie_fill_dense(gen.dev.h, int(cap), _ffi.ptr(A)))
    return A
