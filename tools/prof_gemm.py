"""Run one semiring GEMM shape through the C ABI repeatedly (for ncu / quick
timing).  python tools/prof_gemm.py --M 8192 --N 8192 --K 8192 --op mul,add"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_00618_b200 import native  # noqa: E402

OPS = {"add": 0, "mul": 1, "max": 2, "min": 3}

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--N", type=int, default=8192)
ap.add_argument("--K", type=int, default=8192)
ap.add_argument("--op", default="mul,add")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--normal", action="store_true", help="standard-normal operands instead of U[-1,1)")
a = ap.parse_args()
native.init(0)
c, r = (OPS[x] for x in a.op.split(","))
torch.manual_seed(0)
A = torch.randn(a.M, a.K, device="cuda") if a.normal else torch.rand(a.M, a.K, device="cuda") * 2 - 1
B = torch.randn(a.K, a.N, device="cuda") if a.normal else torch.rand(a.K, a.N, device="cuda") * 2 - 1
C = torch.empty(a.M, a.N, device="cuda")
d = native.GemmDesc()
d.M, d.N, d.K, d.batch = a.M, a.N, a.K, 1
d.A, d.sa_m, d.sa_k = A.data_ptr(), a.K, 1
d.B, d.sb_k, d.sb_n = B.data_ptr(), a.N, 1
d.C, d.sc_m, d.sc_n = C.data_ptr(), a.N, 1
d.combine, d.reduce, d.beta = c, r, 1.0
d.n_epi = 1
d.epi[0].combine, d.epi[0].reduce, d.epi[0].beta = -1, r, 1.0
d.algo, d.split_k, d.tile_m = a.algo, a.split, a.tile
s = torch.cuda.current_stream()
for _ in range(2):
    native.semiring_gemm(d, s.cuda_stream)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
for i in range(a.reps):
    ev[2 * i].record(s)
    native.semiring_gemm(d, s.cuda_stream)
    ev[2 * i + 1].record(s)
torch.cuda.synchronize()
ts = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(a.reps)]
fl = 2.0 * a.M * a.N * a.K
print(f"{a.op} {a.M}x{a.N}x{a.K}: min {min(ts):.3f} ms  {fl / min(ts) / 1e9:.1f} TFLOP/s  "
      f"mean {sum(ts) / len(ts):.3f} ms")
if a.op == "mul,add":
    rows = torch.unique(torch.cat([torch.arange(min(64, a.M)), torch.randint(0, a.M, (64,))])).cuda()
    ref = A[rows].double() @ B.double()
    d = (C[rows].double() - ref).abs()
    err = (d / ref.abs().clamp(min=1)).max().item()
    strict = (d <= 1e-5 + 1e-4 * ref.abs()).double().mean().item()
    print(f"check {len(rows)} rows: ref-metric {err:.3e}  strict-pass {strict:.6f}")
