"""B200-native CBIE fill -> ACA -> H-LU (drop-in for the chebscat hot path).

Host Python mirrors the reference API (Problem, build_hmatrix, solve_direct,
solve_dense); all hot-path arithmetic runs in libcbie.so (hand-written CUDA
for sm_100a) behind the C-ABI in include/cbie.h.  There is no CPU fallback.
"""

from . import errors, geometry, kernels  # noqa: F401

__version__ = "0.1.0"
