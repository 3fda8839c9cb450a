"""B200-native CBIE fill -> ACA -> H-LU (drop-in for the chebscat hot path).

Host Python mirrors the reference API (Problem, build_hmatrix, solve_direct,
solve_dense); all hot-path arithmetic runs in libcbie.so (hand-written CUDA
for sm_100a) behind the C-ABI in include/cbie.h.  There is no CPU fallback.
"""

import os as _os

# The H-LU executor runs ~20 concurrent streams (csrc/hlu.cu, StreamPool); with the
# default 8 hardware work queues unrelated streams share a queue and serialise.
# Read when the CUDA context is created, so it must be set before the first CUDA call.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import errors, geometry, kernels  # noqa: F401,E402

__version__ = "0.1.0"
