"""Multi-GPU plumbing of the H-matrix fill and H-LU: one process
per GPU, torch.distributed only to hand the NCCL unique id to every rank; the
shard exchange (csrc/shard.cu) and the block-row-distributed H-LU exchanges
(csrc/hlu_dist.cuh) are NCCL calls inside libcbie.

The reference parallelises the fill with a ThreadPoolExecutor over leaves
(hmatrix.py:217-219); here the leaves are partitioned over processes by the
same deterministic LPT rule on every rank (partition_lpt)."""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _ffi


def partition_lpt(cost, world: int) -> np.ndarray:
    """Owner of every work item: largest cost first, each to the least-loaded rank
    (ties to the lowest rank).  Host-only (cbie_partition_lpt)."""
    lib = _ffi.load()
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
    owner = np.empty(c.shape[0], np.int32)
    lib.cbie_partition_lpt(_ffi.ptr(c), int(c.shape[0]), int(world), _ffi.ptr(owner))
    return owner


def init_nccl(gen, rank: int, world: int, group=None) -> None:
    """Create the context's NCCL communicator: rank 0 draws the unique id, the
    default torch.distributed group (any backend) carries it to every rank."""
    import torch.distributed as dist
    lib = gen.dev.lib
    buf = ct.create_string_buffer(128)
    if rank == 0:
        _ffi.check(lib.cbie_nccl_unique_id(buf, 128))
    obj = [bytes(buf.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    gen.dev.check(lib.cbie_dist_init(gen.dev.h, obj[0], int(rank), int(world)))


def finalize(gen) -> None:
    gen.dev.lib.cbie_dist_finalize(gen.dev.h)


def hlu_factor_distributed(H, tol: float):
    """Block-row-distributed H-LU (cbie_hlu_factor_dist): every rank passes the
    same complete H-matrix and gets the complete factors back."""
    from .hmatrix import HLUFactors
    return HLUFactors(H, tol, distributed=True)


def hlu_dist_plan(points, C: int, n_leaf: int, eta: float, world: int):
    """Host-only distributed H-LU plan of the block structure of `points` (no GPU):
    (stats dict, leaf owner array) -- cbie_hlu_dist_plan_host."""
    lib = _ffi.load()
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    st = np.zeros(11, np.int64)
    args = (_ffi.ptr(pts), int(pts.shape[0]), int(C), int(n_leaf), float(eta), int(world), _ffi.ptr(st))
    _ffi.check(lib.cbie_hlu_dist_plan_host(*args, None))
    owner = np.full(int(st[10]), -1, np.int32)
    _ffi.check(lib.cbie_hlu_dist_plan_host(*args, _ffi.ptr(owner)))
    keys = ("tasks", "messages", "xfer_buffers", "xfer_elems", "conflicts", "levels", "row_level",
            "tasks_min", "tasks_max", "final_elems", "leaves")
    return dict(zip(keys, (int(v) for v in st))), owner


def shard_layout(m, n, adm, owner, info, world: int):
    """Host-only exchange layout of the sharded fill (cbie_shard_layout_host, the function
    csrc/shard.cu's exchange uses): (leaf offsets [nleaf][3], ranges [world][4], total)."""
    lib = _ffi.load()
    m = np.ascontiguousarray(m, np.int32)
    n = np.ascontiguousarray(n, np.int32)
    adm = np.ascontiguousarray(adm, np.uint8)
    owner = np.ascontiguousarray(owner, np.int32)
    info = np.ascontiguousarray(info, np.int32)
    off = np.empty((m.size, 3), np.int64)
    rng = np.empty((world, 4), np.int64)
    tot = ct.c_int64()
    _ffi.check(lib.cbie_shard_layout_host(int(m.size), _ffi.ptr(m), _ffi.ptr(n), _ffi.ptr(adm), _ffi.ptr(owner),
                                          _ffi.ptr(info), int(world), _ffi.ptr(off), _ffi.ptr(rng), ct.byref(tot)))
    return off, rng, int(tot.value)
