"""CPU baseline workload for bench.py (oracle = test/baseline infrastructure only).

A bounded, projected measurement of the oracle (numpy restatement of the
reference) on config 2 -- the full run takes ~12 min of CPU, so
each step times a sample and projects it to the whole configuration:

  fill  = classification of every (point, patch) pair (timed in full)
        + stratified leaf sample: per stratum (dense / admissible x leaf size)
          ``per_stratum`` seeded leaves are filled through the canonical pair
          blocks / ACA+recompression and timed; mean x stratum count
  H-LU  = recursive H-LU of the leading diagonal H-blocks at tree levels L and
          L+1 (their leaves filled for real), extrapolated to the root with the
          measured growth exponent:  T_root = T_L * (T_L / T_{L+1})^L

The result is reported as unknowns/s = N / (fill + H-LU) of the projection.
"""

from __future__ import annotations

import copy
import math
import os
import time
from collections import defaultdict

import numpy as np

from . import hcompress as hc
from . import hfactor as hf
from . import nearfield as nf
from . import pipeline as pl


def _diag(node, level):
    for _ in range(level):
        if node.kind != "H":
            break
        node = node.kids[0][0]
    return node


def step(cfg: int = 2, level: int = 3, per_stratum: int = 3, seed: int = 7):
    """Returns (N, projected seconds, detail dict)."""
    cs = pl.case(cfg)
    disc = cs.disc()
    gen = nf.Scaled(disc)
    H = hc.HMat(disc.pos, disc.C, cs.n_leaf, cs.eta)
    lv = hc.leaves(H.root)
    t0 = time.perf_counter()
    disc.classify_all()
    t_class = time.perf_counter() - t0
    # stratified leaf sample over the whole matrix
    strata = defaultdict(list)
    for i, b in enumerate(lv):
        strata[(b.kind, (b.r.hi - b.r.lo) * H.C)].append(i)
    rng = np.random.default_rng(seed)
    t_fill = t_class
    for key, ids in sorted(strata.items()):
        pick = rng.choice(len(ids), size=min(per_stratum, len(ids)), replace=False)
        ts = []
        for p in pick:
            t = time.perf_counter()
            H.fill(gen, cs.aca_tol, sample=[ids[p]])
            ts.append(time.perf_counter() - t)
        t_fill += len(ids) * float(np.mean(ts))
    # H-LU growth from two nested diagonal blocks
    sub = _diag(H.root, level)
    sub_ids = {id(b) for b in hc.leaves(sub)}
    H.fill(gen, cs.aca_tol, sample=[i for i, b in enumerate(lv) if id(b) in sub_ids])
    t = time.perf_counter()
    hf._factor(copy.deepcopy(sub), H.C, cs.aca_tol)
    t_l = time.perf_counter() - t
    t = time.perf_counter()
    hf._factor(copy.deepcopy(sub.kids[0][0]), H.C, cs.aca_tol)
    t_l1 = time.perf_counter() - t
    growth = max(t_l / max(t_l1, 1e-9), 1.0)
    t_hlu = t_l * growth ** level
    detail = {"classify_s": t_class, "fill_projected_s": t_fill, "hlu_level_s": t_l,
              "hlu_level_plus1_s": t_l1, "hlu_growth_per_level": growth,
              "hlu_projected_s": t_hlu}
    return H.N, t_fill + t_hlu, detail


def describe(cfg=2, level=3, per_stratum=3):
    return (f"oracle (numpy port), config {cfg}, projected from a bounded sample: full "
            f"classification + {per_stratum} seeded leaves per (kind, size) stratum scaled by the "
            f"stratum counts; H-LU of the level-{level} and level-{level + 1} leading diagonal "
            f"H-blocks extrapolated to the root by their growth ratio; "
            f"OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS', 'default')}")


def _calibration(cfg):
    import json
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "calibration.json")
    cal = json.load(open(path))
    key = str(cfg) if str(cfg) in cal else "2"
    c = cal[key]
    return key, c["ref_fill_s"] / c["port_fill_projected_s"], c["ref_factor_s"] / c["port_hlu_projected_s"]


def calibrated_step(cfg: int = 2, level: int = 3):
    """One bounded sample of the port (``step``) scaled per phase by the measured ratio of
    the reference's full run to the port's projection (oracle/calibration.json), i.e. an
    estimate of the reference's own fill + H-LU time on this host.  Returns
    (N, seconds, detail)."""
    t0 = time.perf_counter()
    n, sec, det = step(cfg, level)
    wall = time.perf_counter() - t0
    key, kf, kh = _calibration(cfg)
    fill = det["fill_projected_s"] * kf
    hlu = det["hlu_projected_s"] * kh
    det = dict(det, calibration_config=int(key), k_fill=kf, k_hlu=kh, fill_s=fill, hlu_s=hlu,
               sample_wall_s=wall,
               sample=describe(cfg, level) + f"; calibrated per phase to the reference's measured full "
               f"run of config {key} (oracle/calibration.json: fill x{kf:.3f}, H-LU x{kh:.3f})")
    return n, fill + hlu, det
