"""Exception hierarchy of the drop-in (same names as the reference, errors.py:1-73).

C-ABI status codes (include/cbie.h) map onto these in _ffi.check().
"""


class ChebscatError(Exception):
    """Base class for all package-specific errors."""


class DegeneratePatch(ChebscatError):
    pass


class DimensionError(ChebscatError):
    pass


class SingularPoint(ChebscatError):
    pass


class RankOverflow(ChebscatError):
    pass


class SingularDiagonal(ChebscatError):
    pass


class CapExceeded(ChebscatError):
    pass


class UnsupportedExcitation(ChebscatError):
    pass


class NativeUnavailable(RuntimeError):
    """libcbie.so is missing or no CUDA device is visible: there is no CPU fallback."""
