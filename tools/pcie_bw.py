"""Pinned host<->device copy bandwidth through the library's copy calls."""
import os
import sys
import time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_00618_b200 import native  # noqa: E402
native.init(0)
n = 1 << 28   # 1 GiB of f32
h = native.PinnedBuffer((n,))
d = native.DeviceBuffer(4 * n)
h.array[:] = 1.0
for name, fn in (("h2d", lambda: native.h2d(d.ptr, h.array.ctypes.data, 4 * n, 0)),
                 ("d2h", lambda: native.d2h(h.array.ctypes.data, d.ptr, 4 * n, 0))):
    fn(); native.sync(0)
    t = time.perf_counter()
    for _ in range(3):
        fn()
    native.sync(0)
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {4 * n / dt / 1e9:.1f} GB/s")
# pitched: 8 column blocks of a 16384 x 16384 f32 matrix (8 KiB rows)
K = N = 16384
w = N // 8
t = time.perf_counter()
for c0 in range(0, N, w):
    native.h2d_2d(d.ptr + 4 * c0, 4 * N, h.array.ctypes.data + 4 * c0, 4 * N, 4 * w, K, 0)
native.sync(0)
dt = time.perf_counter() - t
print(f"h2d_2d (8 column blocks, 8 KiB rows): {4 * K * N / dt / 1e9:.1f} GB/s")
# full duplex: 1 GiB up and 1 GiB down at the same time on two streams
h2 = native.PinnedBuffer((n,))
d2 = native.DeviceBuffer(4 * n)
s1, s2 = native.Stream(), native.Stream()
for rep in range(2):
    native.sync(0)
    t = time.perf_counter()
    native.h2d(d.ptr, h.array.ctypes.data, 4 * n, s1.handle)
    native.d2h(h2.array.ctypes.data, d2.ptr, 4 * n, s2.handle)
    s1.sync(); s2.sync()
    dt = time.perf_counter() - t
print(f"duplex (1 GiB each way concurrently): {2 * 4 * n / dt / 1e9:.1f} GB/s aggregate, {dt * 1e3:.1f} ms")
