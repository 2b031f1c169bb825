"""Graph-replay timing (L2 flushed between steps, like bench.py) of one GEMM
shape over split-K / tile variants: picks the small-GEMM policy."""
import itertools
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_00618_b200 import native  # noqa: E402

native.init(0)
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 256, 256)))
op = sys.argv[4] if len(sys.argv) > 4 else "mul,add"
OPS = {"add": 0, "mul": 1, "max": 2, "min": 3}
c, r = (OPS[x] for x in op.split(","))
A = torch.rand(M, K, device="cuda")
B = torch.rand(K, N, device="cuda")
C = torch.empty(M, N, device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
res = []
for split, tile in itertools.product([0, 1, 2, 4, 8, 16], [0, 64, 128]):
    d = native.GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, 1
    d.A, d.sa_m, d.sa_k = A.data_ptr(), K, 1
    d.B, d.sb_k, d.sb_n = B.data_ptr(), N, 1
    d.C, d.sc_m, d.sc_n = C.data_ptr(), N, 1
    d.combine, d.reduce, d.beta = c, r, 1.0
    d.algo, d.split_k, d.tile_m = 1, split, tile
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        native.semiring_gemm(d, s.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            native.semiring_gemm(d, s.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.append((min(ts), split, tile))
    print(f"split={split:2d} tile={tile:3d}: {min(ts) * 1e3:.1f} us")
print("best", min(res))
