"""Host-side copy costs on the GPU box: cudaHostRegister / Unregister of a
1 GiB numpy array, pageable vs pinned H2D, multi-threaded memcpy bandwidth."""
import time
import threading

import numpy as np
import torch

n = 1 << 28   # 1 GiB of f32
a = np.ones(n, np.float32)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
cr = torch.cuda.cudart()
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    dev.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms (rc {r}), H2D registered {1e3*(t2-t1):.1f} ms, unregister {1e3*(t3-t2):.1f} ms")
t0 = time.perf_counter()
dev.copy_(torch.from_numpy(a))
torch.cuda.synchronize()
print(f"H2D pageable {1e3*(time.perf_counter()-t0):.1f} ms")
b = np.empty_like(a)
for th in (1, 4, 8, 16):
    chunks = np.array_split(np.arange(n), th)
    def work(c):
        np.copyto(b[c[0]:c[-1] + 1], a[c[0]:c[-1] + 1])
    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(c,)) for c in chunks]
    [t.start() for t in ts]
    [t.join() for t in ts]
    dt = time.perf_counter() - t0
    print(f"memcpy {th} threads: {a.nbytes / dt / 1e9:.1f} GB/s")
