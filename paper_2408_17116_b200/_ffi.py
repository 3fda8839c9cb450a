"""ctypes binding of libcbie.so (include/cbie.h).  No CPU fallback: if the
library or a CUDA device is missing every entry point raises NativeUnavailable."""

from __future__ import annotations

import ctypes as ct
import os
import threading

import numpy as np

from . import errors

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcbie.so")
_lib = None
_lock = threading.Lock()


class C128(ct.Structure):
    _fields_ = [("re", ct.c_double), ("im", ct.c_double)]


def c128(z) -> C128:
    z = complex(z)
    return C128(z.real, z.imag)


P = ct.c_void_p
I64P = ct.POINTER(ct.c_int64)

_SIGS = {
    "cbie_create": (ct.c_int, [ct.c_int, ct.POINTER(P)]),
    "cbie_destroy": (None, [P]),
    "cbie_last_error": (ct.c_char_p, [P]),
    "cbie_launch_count": (ct.c_int64, []),
    "cbie_stream": (ct.c_void_p, [P]),
    "cbie_set_geometry": (ct.c_int, [P, ct.c_int, ct.c_int, ct.c_int, P, P, P, P, P]),
    "cbie_node_frames": (ct.c_int, [P, P, P, P, P]),
    "cbie_set_formulation": (ct.c_int, [P, ct.c_int, ct.c_double, C128, C128, C128, C128, C128,
                                        C128, ct.c_double, ct.c_int, ct.c_int, P, P]),
    "cbie_classify": (ct.c_int, [P, I64P, I64P, I64P]),
    "cbie_export_classification": (ct.c_int, [P, ct.c_int64, P, P, P, P, P, P]),
    "cbie_pair_block": (ct.c_int, [P, ct.c_int64, ct.c_int, P]),
    "cbie_fill_block": (ct.c_int, [P, P, ct.c_int64, P, ct.c_int64, ct.c_int, P]),
    "cbie_fill_dense": (ct.c_int, [P, ct.c_int64, P]),
    "cbie_dense_solve": (ct.c_int, [P, ct.c_int64, P, ct.c_int, P, ct.POINTER(ct.c_double), P, P]),
    "cbie_hmatrix_build": (ct.c_int, [P, ct.c_int, ct.c_double, ct.c_double, ct.POINTER(P)]),
    "cbie_hmatrix_destroy": (None, [P]),
    "cbie_hmatrix_offload": (ct.c_int, [P]),
    "cbie_hmatrix_layout": (ct.c_int, [P, ct.c_int64, ct.c_int, ct.c_int, ct.c_double, P, P, I64P]),
    "cbie_hmatrix_import": (ct.c_int, [P, P, ct.c_int64, ct.c_int, ct.c_int, ct.c_double, ct.c_double, P,
                                       ct.POINTER(P)]),
    "cbie_hmatrix_tree": (ct.c_int, [P, P, P, I64P]),
    "cbie_hmatrix_leaf": (ct.c_int, [P, ct.c_int64, ct.POINTER(ct.c_int), ct.POINTER(ct.c_int), P, P]),
    "cbie_hmatvec": (ct.c_int, [P, P, P, ct.c_int]),
    "cbie_hlu_factor": (ct.c_int, [P, ct.c_double, ct.POINTER(P)]),
    "cbie_hlu_destroy": (None, [P]),
    "cbie_far_field_sums": (ct.c_int, [P, P, ct.c_int, P, ct.c_int, ct.c_double, P]),
    "cbie_gmres": (ct.c_int, [P, P, ct.c_double, ct.c_int, ct.c_int, P, ct.POINTER(ct.c_int),
                              ct.POINTER(ct.c_double), ct.POINTER(ct.c_int)]),
    "cbie_hlu_dist_plan_host": (ct.c_int, [P, ct.c_int64, ct.c_int, ct.c_int, ct.c_double, ct.c_int, P, P]),
    "cbie_hlu_factor_dist": (ct.c_int, [P, ct.c_double, ct.POINTER(P)]),
    "cbie_hlu_factor_emulated": (ct.c_int, [P, ct.c_double, ct.c_int, ct.POINTER(P)]),
    "cbie_hlu_leaf": (ct.c_int, [P, ct.c_int64, ct.POINTER(ct.c_int), ct.POINTER(ct.c_int), P, P, P]),
    "cbie_hlu_solve": (ct.c_int, [P, P, P, ct.c_int]),
    "cbie_lowrank_truncate": (ct.c_int, [P, P, ct.c_int, ct.c_int, P, ct.c_int, ct.c_double,
                                         ct.POINTER(ct.c_int), P, P]),
    "cbie_trunc_bench": (ct.c_int, [P, ct.c_int, ct.c_int, ct.c_int, ct.c_int, ct.c_int, ct.c_double,
                                    ct.c_int, ct.c_int, P, P, P]),
    "cbie_stats_json": (ct.c_int, [P, ct.c_int, ct.c_char_p, ct.c_size_t]),
    "cbie_partition_lpt": (None, [P, ct.c_int64, ct.c_int, P]),
    "cbie_shard_layout_host": (ct.c_int, [ct.c_int, P, P, P, P, P, ct.c_int, P, P, I64P]),
    "cbie_nccl_unique_id": (ct.c_int, [ct.c_char_p, ct.c_int]),
    "cbie_dist_init": (ct.c_int, [P, ct.c_char_p, ct.c_int, ct.c_int]),
    "cbie_dist_finalize": (None, [P]),
    "cbie_hmatrix_build_shard": (ct.c_int, [P, ct.c_int, ct.c_double, ct.c_double, ct.c_int, ct.c_int,
                                            ct.c_int, ct.POINTER(P)]),
}

EXPORTED = tuple(_SIGS)


def load(path: str | None = None):
    """Load libcbie.so (in-tree build).  Raises NativeUnavailable if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or _LIB_PATH
        if not os.path.exists(p):
            raise errors.NativeUnavailable(
                f"{p} not built; run paper_2408_17116_b200.build.build() (no CPU fallback)")
        # torch (plumbing for streams / torch.distributed) bundles a newer NCCL under
        # the same soname; load it first so libcbie binds to that one and a later
        # `import torch` does not resolve its NCCL symbols against an older library
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        lib = ct.CDLL(p)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


_CODE = {
    1: errors.SingularDiagonal,
    2: errors.DegeneratePatch,
    3: errors.SingularPoint,
    4: errors.CapExceeded,
    5: errors.RankOverflow,
}


def check(rc: int, ctx=None):
    if rc == 0:
        return
    msg = ""
    if ctx is not None:
        msg = (_lib.cbie_last_error(ctx) or b"").decode()
    exc = _CODE.get(rc)
    if exc is not None:
        raise exc(msg)
    if rc in (10, 12) and "no CUDA-capable device" in msg:
        raise errors.NativeUnavailable(msg)
    raise RuntimeError(f"libcbie error {rc}: {msg}")


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


def stats(handle, which: int) -> dict:
    import json
    buf = ct.create_string_buffer(1 << 16)
    check(_lib.cbie_stats_json(handle, which, buf, len(buf)))
    return json.loads(buf.value.decode() or "{}")
