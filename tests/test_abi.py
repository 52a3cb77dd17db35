"""The C-ABI boundary (CPU): libofl.so loads without a GPU and exports every
entry point include/ofl.h declares, with the prototypes the ctypes layer
attaches; the status codes match the reference's wire codes.  No compute
call is made here."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from paper_1810_11482_b200 import _native, errors

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "ofl.h")


def declared() -> set:
    text = open(HEADER).read()
    return set(re.findall(r"^(?:int|uint64_t|const char\*|void\*)\s+(ofl_\w+)\(", text, re.M))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    names = declared()
    assert len(names) >= 40
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ofl_\w+)", out))
    assert names <= exported, names - exported


def test_ctypes_prototypes_cover_header():
    assert declared() == set(_native.EXPORTED)


def test_status_codes_match_reference_wire_codes():
    text = open(HEADER).read()
    codes = dict(re.findall(r"#define (OFL_ERR_\w+) (\d+)", text))
    assert int(codes["OFL_ERR_UNKNOWN_GID"]) == errors.ERR_UNKNOWN_GID == 1
    assert int(codes["OFL_ERR_BAD_ARGS"]) == errors.ERR_BAD_ARGS == 2
    assert int(codes["OFL_ERR_COMPILE"]) == errors.ERR_COMPILE == 3
    assert int(codes["OFL_ERR_OOB_ACCESS"]) == errors.ERR_OOB_ACCESS == 4
    assert int(codes["OFL_ERR_INTERNAL"]) == errors.ERR_INTERNAL == 5


def test_abi_version_and_null_stream_rejected():
    lib = _native.load()
    assert lib.ofl_abi_version() == 1
    t = ctypes.c_uint64()
    assert lib.ofl_h2d(None, None, None, 0, ctypes.byref(t)) == _native.OFL_ERR_BAD_ARGS
    assert "null stream" in _native.last_error()


def test_status_maps_to_exception_types():
    assert isinstance(_native.error_for(_native.OFL_ERR_OOB_ACCESS), errors.OobAccessError)
    assert isinstance(_native.error_for(_native.OFL_ERR_OOM), errors.OutOfMemoryError)
    assert isinstance(_native.error_for(_native.OFL_ERR_CUDA), errors.InternalError)


def test_no_cpu_fallback_without_gpu():
    """The product path fails loudly when no CUDA device is usable."""
    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_1810_11482_b200 import Runtime

    with pytest.raises(errors.InternalError, match="no CUDA device"):
        Runtime()


def test_product_package_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_1810_11482_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
