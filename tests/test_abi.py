"""The C ABI library loads and exports every symbol include/lsb.h declares;
the ctypes struct mirrors match the C layout.  No kernel runs (CPU only)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2205_00618_b200 import native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "lsb.h")


def declared() -> set[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:int|int64_t)\s+(lsb_\w+)\s*\(", src, flags=re.M))


def test_header_declares_entry_points():
    names = declared()
    for n in ("lsb_init", "lsb_semiring_gemm", "lsb_conv2d_nchw", "lsb_affine_nest",
              "lsb_last_error", "lsb_device_alloc", "lsb_memcpy_h2d"):
        assert n in names


def test_library_exports_every_declared_symbol():
    L = native.lib()
    for name in sorted(declared()):
        assert hasattr(L, name), name
    assert set(native.EXPORTS) == declared()


def test_struct_layouts_match():
    L = native.lib()
    for i, s in enumerate(native.STRUCTS):
        assert L.lsb_sizeof(i) == ctypes.sizeof(s), s.__name__


def test_abi_version_and_error_path_without_gpu():
    L = native.lib()
    assert L.lsb_abi_version() == native.ABI_VERSION
    # a null descriptor is rejected before touching the device
    rc = L.lsb_semiring_gemm(None, None)
    assert rc == -1
    assert "null" in native.last_error()


def test_invalid_descriptor_rejected():
    d = native.GemmDesc()
    d.M = d.N = d.K = 4
    d.batch = 1
    d.combine, d.reduce = 7, 0
    with pytest.raises(native.NativeError, match="operator pair"):
        native.semiring_gemm(d)


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(native, "_LIB", None)
    monkeypatch.setattr(native, "LIB_PATH", "/nonexistent/liblsb.so")
    with pytest.raises(native.NativeError, match="no CPU fallback"):
        native.lib()


def test_nccl_unique_id_without_gpu():
    """lsb_nccl_unique_id resolves NCCL at run time (dlopen) and needs no GPU;
    bad communicator arguments are rejected before NCCL is touched."""
    a, b = native.nccl_unique_id(), native.nccl_unique_id()
    assert len(a) == native.NCCL_ID_BYTES and a != b
    with pytest.raises(native.NativeError, match="bad communicator"):
        native.NcclComm(2, 2, a)
    rc = native.lib().lsb_allgather_rows(None, None, None, 4, None)
    assert rc < 0 and "bad gather" in native.last_error()
