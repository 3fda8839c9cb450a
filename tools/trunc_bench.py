"""Gram-path recompression micro-benchmark (cbie_trunc_bench): per (m, n, k) shape,
nprob problems of numerical rank ~r in one launch; prints launch ms, per-problem
phase cycles (CBIE_PROFILE counters) and the kept ranks."""
import ctypes as ct
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2408_17116_b200 import _ffi  # noqa: E402
from paper_2408_17116_b200.assembly import Device  # noqa: E402

d = Device(0)
shapes = [(256, 256, 32, 16, 148), (256, 256, 64, 30, 148), (384, 384, 64, 30, 148), (768, 768, 64, 30, 64),
          (1536, 1536, 64, 40, 32), (1536, 1536, 48, 30, 32), (768, 768, 100, 50, 32), (1536, 1536, 100, 50, 32)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
names = ["gram", "core", "svd", "apply"]
gnames = ["pchol_uv", "core_H", "pchol_H", "gp", "w_vhat", "trisolve_u", "apply_u"]
for (m, n, k, r, npb, *rest) in shapes:
    cs = rest[0] if rest else 1
    ms = ct.c_float()
    prof = np.zeros(32, np.uint64)
    rk = np.zeros(npb, np.int32)
    d.check(d.lib.cbie_trunc_bench(d.h, m, n, k, r, npb, 1e-4, cs, 5, ct.byref(ms), _ffi.ptr(prof), _ffi.ptr(rk)))
    cnt = max(int(prof[14]), 1)
    out = {"m": m, "n": n, "k": k, "nprob": npb, "csize": cs, "ms": round(ms.value, 4),
           "rank": int(np.median(rk)),
           "cyc_total": int(prof[15]) // cnt}
    out.update({nm: int(prof[i]) // cnt for i, nm in enumerate(names)})
    out.update({nm: int(prof[16 + i]) // cnt for i, nm in enumerate(gnames)})
    out["flops_per_prob"] = 8.0 * (m + n) * k * k / 2
    print(json.dumps(out), flush=True)
