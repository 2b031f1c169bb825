import os, sys, json
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tests")]
import common
from paper_2205_00618_b200 import backend, native
native.setenv("LSB_GEMM_ALGO", "tf32x3")
idx = json.load(open(os.path.join(R, "tests/golden/index.json")))
c = [c for c in idx["cases"] if c["name"] == "semiring_mul_add"][0]
gj = common.graph_json(c["graph"])
ins, ref, _ = common.case_data(c)
k = backend.compile_graph(gj)
for trial in range(2):
    got = {s: np.array(b, copy=True) for s, b in ins.items()}
    backend.execute(k, got)
    g = got[2].reshape(37, 53).astype(np.float64); r = ref[2].reshape(37, 53)
    d = np.abs(g - r)
    print("metric", d.max() / np.abs(r).max(), "bad elems", int((d > 1e-3).sum()), np.argwhere(d > 1e-3)[:10].tolist())
A = ins[0].astype(np.float64); B = ins[1].astype(np.float64)
print("ref vs A@B", np.abs(A @ B - r).max())
print("slots", {s: (a.shape, a.dtype, a.flags['C_CONTIGUOUS']) for s, a in ins.items()})
