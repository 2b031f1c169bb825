"""C3 through bench.py's per-config path (CUDA graph per step, L2 flushed
between steps) for each conv kernel: python tools/bench_c3.py [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2205_00618_b200 import native  # noqa: E402

native.init(0)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for algo in ("tf32x3_nhwc", "tf32x3_planar"):
    native.setenv("LSB_GEMM_ALGO", algo)
    r = bench.gpu_config_run("C3", steps, 5, torch, 0, 1, flush_l2=True, want_e2e=False)
    g = bench.FLOPS["C3"] / (r["ms_mean"] * 1e-3) / 1e12
    print(f"{algo:12s} step {r['ms_mean'] * 1e3:7.2f} us  min {r['ms_min'] * 1e3:7.2f} us  kernel {r['kernel_ms'] * 1e3:7.2f} us"
          f"  {g:6.1f} TF/s  frac(274) {g / 274.03:.3f}  parity {r['parity'].get('strict_pass')}")
native.setenv("LSB_GEMM_ALGO", None)
