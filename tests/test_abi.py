"""CPU-side checks of the drop-in boundary: libcbie.so builds, loads, and exports
every symbol include/cbie.h declares (no compute calls: no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2408_17116_b200", "libcbie.so")


def declared():
    txt = open(os.path.join(ROOT, "include", "cbie.h")).read()
    return sorted(set(re.findall(r"\b(cbie_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2408_17116_b200 import build
    build.build()
    import torch  # noqa: F401  (torch's NCCL first, as _ffi.load does)
    return ctypes.CDLL(LIB)


def test_header_declares_the_documented_boundary():
    names = declared()
    for must in ("cbie_create", "cbie_classify", "cbie_fill_block", "cbie_hmatrix_build",
                 "cbie_hlu_factor", "cbie_hlu_solve", "cbie_hmatvec"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ffi_signatures_cover_header(lib):
    from paper_2408_17116_b200 import _ffi
    assert set(_ffi.EXPORTED) == set(declared())
    _ffi.load()


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2408_17116_b200.assembly import Device
    from paper_2408_17116_b200.errors import NativeUnavailable
    with pytest.raises(NativeUnavailable):
        Device(0)
