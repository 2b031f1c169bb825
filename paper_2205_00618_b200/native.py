"""ctypes binding of liblsb.so (include/lsb.h).

There is no CPU fallback: importing the backend on a machine without the
built library, or calling a kernel without a CUDA device, raises
``NativeError`` loudly (the reference would otherwise silently keep using its
VM, which this backend replaces).
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSB_LIB_PATH") or os.path.join(PKG, "liblsb.so")   # override: A/B builds (experiments)

LSB_MAX_EPI = 4
LSB_MAX_NEST_DIMS = 8
LSB_MAX_NEST_OPERANDS = 4
LSB_MAX_GUARDS = 4
ABI_VERSION = 3

i32, i64, f32, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class NativeError(RuntimeError):
    """liblsb.so is missing, failed to load, or a call returned an error."""


class EpiStage(ctypes.Structure):
    _fields_ = [("combine", i32), ("reduce", i32), ("pre", i32), ("post", i32),
                ("beta", f32), ("alpha", f32),
                ("operand", vp), ("so", i64 * 4),
                ("c_in", vp), ("sc", i64 * 4)]


class GemmDesc(ctypes.Structure):
    _fields_ = [("M", i64), ("N", i64), ("K", i64), ("batch", i64),
                ("A", vp), ("sa_b", i64), ("sa_m", i64), ("sa_k", i64),
                ("B", vp), ("sb_b", i64), ("sb_k", i64), ("sb_n", i64),
                ("C", vp), ("sc_b", i64), ("sc_m", i64), ("sc_n", i64),
                ("combine", i32), ("reduce", i32),
                ("beta", f32), ("beta_in_loop", i32),
                ("n_epi", i32), ("epi", EpiStage * LSB_MAX_EPI),
                ("algo", i32), ("split_k", i32), ("tile_m", i32), ("tile_n", i32),
                ("m_begin", i64), ("m_end", i64),
                ("flags", i32), ("gen", i32),
                ("n_begin", i64), ("n_end", i64)]


GEMM_B_UNCHANGED = 1
GEMM_PREP_A, GEMM_PREP_B, GEMM_PRESPLIT, GEMM_GROW = 2, 4, 8, 16


class ConvDesc(ctypes.Structure):
    _fields_ = [("N", i64), ("C", i64), ("H", i64), ("W", i64),
                ("CO", i64), ("R", i64), ("S", i64), ("HO", i64), ("WO", i64),
                ("stride_h", i64), ("stride_w", i64), ("pad_h", i64), ("pad_w", i64),
                ("dil_h", i64), ("dil_w", i64),
                ("fill", f32),
                ("x", vp), ("sx", i64 * 4),
                ("w", vp), ("sw", i64 * 4),
                ("o", vp), ("so", i64 * 4),
                ("combine", i32), ("reduce", i32),
                ("beta", f32), ("beta_in_loop", i32),
                ("n_epi", i32), ("epi", EpiStage * LSB_MAX_EPI)]


class Affine(ctypes.Structure):
    _fields_ = [("base", i64), ("coeff", i64 * LSB_MAX_NEST_DIMS)]


class NestOperand(ctypes.Structure):
    _fields_ = [("ptr", vp), ("addr", Affine), ("n_guards", i32),
                ("guard", Affine * LSB_MAX_GUARDS), ("guard_size", i64 * LSB_MAX_GUARDS),
                ("fill", f32)]


class NestDesc(ctypes.Structure):
    _fields_ = [("n_out", i32), ("n_red", i32),
                ("extent", i64 * LSB_MAX_NEST_DIMS),
                ("n_operands", i32),
                ("operand", NestOperand * LSB_MAX_NEST_OPERANDS),
                ("out", vp), ("out_addr", Affine),
                ("combine", i32), ("reduce", i32),
                ("beta", f32),
                ("n_epi", i32), ("epi", EpiStage * LSB_MAX_EPI)]


_LIB = None
_LOCK = threading.Lock()
_INIT_DEVICES: set[int] = set()

_SIGS = {
    "lsb_abi_version": ([], ctypes.c_int),
    "lsb_init": ([ctypes.c_int], ctypes.c_int),
    "lsb_last_error": ([ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
    "lsb_reload_env": ([], ctypes.c_int),
    "lsb_device_info": ([ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 4, ctypes.c_int),
    "lsb_device_alloc": ([ctypes.POINTER(vp), ctypes.c_size_t], ctypes.c_int),
    "lsb_device_free": ([vp], ctypes.c_int),
    "lsb_host_alloc": ([ctypes.POINTER(vp), ctypes.c_size_t], ctypes.c_int),
    "lsb_host_free": ([vp], ctypes.c_int),
    "lsb_memcpy_h2d": ([vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
    "lsb_memcpy_d2h": ([vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
    "lsb_memcpy_d2d": ([vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
    "lsb_memcpy_h2d_2d": ([vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, vp],
                          ctypes.c_int),
    "lsb_memcpy_d2h_2d": ([vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, vp],
                          ctypes.c_int),
    "lsb_stream_sync": ([vp], ctypes.c_int),
    "lsb_stage_h2d_2d": ([vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, vp],
                         ctypes.c_int),
    "lsb_stage_d2h_2d": ([vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, vp],
                         ctypes.c_int),
    "lsb_stage_wait": ([], ctypes.c_int),
    "lsb_host_is_pinned": ([vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "lsb_last_gemm_launch": ([ctypes.POINTER(ctypes.c_int)] * 4, ctypes.c_int),
    "lsb_last_conv_kernel": ([ctypes.POINTER(ctypes.c_int)] * 2, ctypes.c_int),
    "lsb_last_nest_kernel": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "lsb_nccl_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "lsb_nccl_init": ([ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(vp)], ctypes.c_int),
    "lsb_nccl_destroy": ([vp], ctypes.c_int),
    "lsb_allgather_rows": ([vp, vp, vp, i64, vp], ctypes.c_int),
    "lsb_stream_create": ([ctypes.POINTER(vp)], ctypes.c_int),
    "lsb_stream_destroy": ([vp], ctypes.c_int),
    "lsb_event_create": ([ctypes.POINTER(vp)], ctypes.c_int),
    "lsb_event_destroy": ([vp], ctypes.c_int),
    "lsb_event_record": ([vp, vp], ctypes.c_int),
    "lsb_stream_wait_event": ([vp, vp], ctypes.c_int),
    "lsb_semiring_gemm": ([ctypes.POINTER(GemmDesc), vp], ctypes.c_int),
    "lsb_gemm_algo": ([ctypes.POINTER(GemmDesc)], ctypes.c_int),
    "lsb_conv2d_nchw": ([ctypes.POINTER(ConvDesc), vp], ctypes.c_int),
    "lsb_affine_nest": ([ctypes.POINTER(NestDesc), vp], ctypes.c_int),
    "lsb_launch_count": ([ctypes.c_int], ctypes.c_int64),
    "lsb_sizeof": ([ctypes.c_int], ctypes.c_int64),
    "lsb_profile": ([ctypes.c_int], ctypes.c_int),
    "lsb_last_kernel_ms": ([ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
}

#: ctypes mirrors of the lsb.h structs, in lsb_sizeof() order
STRUCTS = (GemmDesc, ConvDesc, NestDesc, EpiStage)

#: every symbol include/lsb.h declares (checked by tests/test_abi.py)
EXPORTS = tuple(_SIGS)


def lib():
    """Load liblsb.so once; raise NativeError if it is absent or stale."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} not built: run `python -m paper_2205_00618_b200.build` "
                "(there is no CPU fallback)")
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as e:
            raise NativeError(f"cannot load {LIB_PATH}: {e}") from None
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.lsb_abi_version() != ABI_VERSION:
            raise NativeError("liblsb.so ABI version mismatch; rebuild it")
        _LIB = L
    return _LIB


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    lib().lsb_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed ({rc}): {last_error()}")


def init(device: int = 0) -> None:
    if device in _INIT_DEVICES:
        return
    check(lib().lsb_init(device), f"lsb_init({device})")
    _INIT_DEVICES.add(device)


def reload_env() -> None:
    """Make liblsb re-read its LSB_* environment knobs (read once otherwise)."""
    check(lib().lsb_reload_env(), "lsb_reload_env")


def setenv(name: str, value: str | None) -> None:
    """Set (or with None unset) an LSB_* knob and reload the library's copy."""
    if value is None:
        os.environ.pop(name, None)
    else:
        os.environ[name] = value
    reload_env()


def device_info(device: int = 0) -> dict:
    sm, ma, mi, clk = (ctypes.c_int() for _ in range(4))
    check(lib().lsb_device_info(device, ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi),
                                ctypes.byref(clk)), "lsb_device_info")
    return {"sm_count": sm.value, "cc": (ma.value, mi.value), "clock_khz": clk.value}


def profile(enable: bool) -> None:
    check(lib().lsb_profile(1 if enable else 0), "lsb_profile")


def last_kernel_ms() -> float:
    v = ctypes.c_float()
    check(lib().lsb_last_kernel_ms(ctypes.byref(v)), "lsb_last_kernel_ms")
    return float(v.value)


def launch_count(reset: bool = False) -> int:
    return int(lib().lsb_launch_count(1 if reset else 0))


class DeviceBuffer:
    """Owned device allocation (freed on close / garbage collection)."""

    def __init__(self, nbytes: int):
        p = vp()
        check(lib().lsb_device_alloc(ctypes.byref(p), max(int(nbytes), 16)), "lsb_device_alloc")
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)

    def close(self) -> None:
        if self.ptr and _LIB is not None:
            _LIB.lsb_device_free(vp(self.ptr))
        self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host allocation exposed as a numpy array."""

    def __init__(self, shape, dtype="float32"):
        import numpy as np
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = vp()
        check(lib().lsb_host_alloc(ctypes.byref(p), max(n, 16)), "lsb_host_alloc")
        self.ptr = int(p.value)
        raw = (ctypes.c_char * max(n, 16)).from_address(self.ptr)
        raw._owner = self      # the array (via its base) keeps the allocation alive
        self.array = np.frombuffer(raw, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def close(self) -> None:
        if self.ptr and _LIB is not None:
            self.array = None
            _LIB.lsb_host_free(vp(self.ptr))
        self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def h2d(dst: int, src: int, nbytes: int, stream: int = 0) -> None:
    check(lib().lsb_memcpy_h2d(vp(dst), vp(src), nbytes, vp(stream)), "lsb_memcpy_h2d")


def h2d_2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream: int = 0) -> None:
    check(lib().lsb_memcpy_h2d_2d(vp(dst), dpitch, vp(src), spitch, width, height, vp(stream)),
          "lsb_memcpy_h2d_2d")


def d2h_2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream: int = 0) -> None:
    check(lib().lsb_memcpy_d2h_2d(vp(dst), dpitch, vp(src), spitch, width, height, vp(stream)),
          "lsb_memcpy_d2h_2d")


def d2h(dst: int, src: int, nbytes: int, stream: int = 0) -> None:
    check(lib().lsb_memcpy_d2h(vp(dst), vp(src), nbytes, vp(stream)), "lsb_memcpy_d2h")


def stage_h2d_2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream: int = 0) -> None:
    check(lib().lsb_stage_h2d_2d(vp(dst), dpitch, vp(src), spitch, width, height, vp(stream)), "lsb_stage_h2d_2d")


def stage_d2h_2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream: int = 0) -> None:
    check(lib().lsb_stage_d2h_2d(vp(dst), dpitch, vp(src), spitch, width, height, vp(stream)), "lsb_stage_d2h_2d")


def stage_wait() -> None:
    check(lib().lsb_stage_wait(), "lsb_stage_wait")


def is_pinned(ptr: int) -> bool:
    v = ctypes.c_int()
    check(lib().lsb_host_is_pinned(vp(ptr), ctypes.byref(v)), "lsb_host_is_pinned")
    return bool(v.value)


def last_gemm_launch() -> dict:
    """Geometry of the last 3xTF32 GEMM launch (tile width, grid, persistent
    units, 2-CTA clusters)."""
    v = [ctypes.c_int() for _ in range(4)]
    check(lib().lsb_last_gemm_launch(*(ctypes.byref(x) for x in v)), "lsb_last_gemm_launch")
    return dict(zip(("bn", "ctas", "units", "pair"), (x.value for x in v)))


def last_nest_kernel() -> int:
    """Which kernel the last affine-nest call launched: 0 general, 1 rows, 2 transpose, 3 vec4, 4 pool, 5 transpose4."""
    k = ctypes.c_int(0)
    check(lib().lsb_last_nest_kernel(ctypes.byref(k)), "lsb_last_nest_kernel")
    return k.value


def last_conv_kernel() -> tuple:
    """(kind, nt) of the last conv launch: kind 0 SIMT, 1 NHWC-copy tensor-core,
    2 planar tensor-core (nt = its pixel tile)."""
    k, nt = ctypes.c_int(), ctypes.c_int()
    check(lib().lsb_last_conv_kernel(ctypes.byref(k), ctypes.byref(nt)), "lsb_last_conv_kernel")
    return k.value, nt.value


def d2d(dst: int, src: int, nbytes: int, stream: int = 0) -> None:
    check(lib().lsb_memcpy_d2d(vp(dst), vp(src), nbytes, vp(stream)), "lsb_memcpy_d2d")


def sync(stream: int = 0) -> None:
    check(lib().lsb_stream_sync(vp(stream)), "lsb_stream_sync")


class Stream:
    """Non-blocking CUDA stream owned by the backend (copy/compute overlap)."""

    def __init__(self):
        p = vp()
        check(lib().lsb_stream_create(ctypes.byref(p)), "lsb_stream_create")
        self.handle = int(p.value)

    def wait(self, event: "Event") -> None:
        check(lib().lsb_stream_wait_event(vp(self.handle), vp(event.handle)), "lsb_stream_wait_event")

    def sync(self) -> None:
        sync(self.handle)

    def __del__(self):
        try:
            if self.handle and _LIB is not None:
                _LIB.lsb_stream_destroy(vp(self.handle))
        except Exception:
            pass


class Event:
    def __init__(self):
        p = vp()
        check(lib().lsb_event_create(ctypes.byref(p)), "lsb_event_create")
        self.handle = int(p.value)

    def record(self, stream: "Stream | int") -> None:
        h = stream.handle if isinstance(stream, Stream) else int(stream)
        check(lib().lsb_event_record(vp(self.handle), vp(h)), "lsb_event_record")

    def __del__(self):
        try:
            if self.handle and _LIB is not None:
                _LIB.lsb_event_destroy(vp(self.handle))
        except Exception:
            pass


def semiring_gemm(desc: GemmDesc, stream: int = 0) -> None:
    check(lib().lsb_semiring_gemm(ctypes.byref(desc), vp(stream)), "lsb_semiring_gemm")


ALGO_NAMES = {0: "auto", 1: "simt", 2: "tf32x3"}


def gemm_algo(desc: GemmDesc) -> str:
    """Algorithm lsb_semiring_gemm picks for ``desc`` (simt | tf32x3)."""
    return ALGO_NAMES.get(int(lib().lsb_gemm_algo(ctypes.byref(desc))), "invalid")


def conv2d_nchw(desc: ConvDesc, stream: int = 0) -> None:
    check(lib().lsb_conv2d_nchw(ctypes.byref(desc), vp(stream)), "lsb_conv2d_nchw")


def affine_nest(desc: NestDesc, stream: int = 0) -> None:
    check(lib().lsb_affine_nest(ctypes.byref(desc), vp(stream)), "lsb_affine_nest")


NCCL_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    check(lib().lsb_nccl_unique_id(buf), "lsb_nccl_unique_id")
    return buf.raw


class NcclComm:
    """NCCL communicator owned by the library (lsb_nccl_init); rank/nranks
    like ncclCommInitRank, the 128-byte id from nccl_unique_id() on one rank."""

    def __init__(self, rank: int, nranks: int, uid: bytes):
        if len(uid) != NCCL_ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        p = vp()
        check(lib().lsb_nccl_init(rank, nranks, uid, ctypes.byref(p)), "lsb_nccl_init")
        self.handle = int(p.value)
        self.rank, self.nranks = rank, nranks

    def allgather_rows(self, send: int, recv: int, count: int, stream: int = 0) -> None:
        check(lib().lsb_allgather_rows(vp(self.handle), vp(send), vp(recv), count, vp(stream)),
              "lsb_allgather_rows")

    def close(self) -> None:
        if self.handle and _LIB is not None:
            _LIB.lsb_nccl_destroy(vp(self.handle))
        self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
