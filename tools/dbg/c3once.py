"""One planar conv launch at C3 (sanitizer / debugging)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2205_00618_b200 import backend, native
native.init(0)
native.setenv("LSB_GEMM_ALGO", os.environ.get("ALGO", "tf32x3_planar"))
k = backend.compile_graph(bench.load_graph("C3"))
host = bench.make_inputs("C3")
bufs = {s: (host[s].copy() if s in host else np.zeros(sh, np.float32)) for s, sh in k.slot_shapes.items()}
backend.execute(k, bufs)
print("ok", float(np.abs(bufs[2]).sum()))
