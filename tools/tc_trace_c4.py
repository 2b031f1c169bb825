"""C4 through run_device with LSB_GEMM_TRACE (a -DLSB_TC_TRACE build via
LSB_LIB_PATH): clock64 stamps of CTA 0 -- ev0[kb] MMA warp got stage kb,
ev1[c] epilogue got chunk c, ev2[c] MMA warp started chunk c (TMEM buffer
free), ev3 milestones."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import common  # noqa: E402
from paper_2205_00618_b200 import backend, native  # noqa: E402

native.init(0)
if len(sys.argv) > 1 and sys.argv[1] == "plain":   # the same GEMM without the bias + ReLU epilogue
    import json
    from paper_2205_00618_b200.shard import shard_graph
    case = next(c for c in common.index()["cases"] if c["name"] == "semiring_mul_add")
    g = json.loads(common.graph_json(case["graph"]))
    for var, n in (("m", 4096), ("k", 1024), ("n", 4096)):
        g = shard_graph(g, n, var)
    k = backend.compile_graph(json.dumps(g))
    ins = common.config_inputs("C4")
    ins = {0: ins[0], 1: ins[1]}
    t = {s: torch.from_numpy(a).cuda() for s, a in ins.items()}
    t[2] = torch.empty(4096, 4096, device="cuda")
    native.setenv("LSB_GEMM_ALGO", "tf32x3")
else:
    k = backend.compile_graph(common.graph_json(common.config("C4")["graph"]))
    ins = common.config_inputs("C4")
    t = {s: torch.from_numpy(a).cuda() for s, a in ins.items()}
    t[3] = torch.empty(4096, 4096, device="cuda")
ptrs = {s: v.data_ptr() for s, v in t.items()}
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    backend.run_device(k, ptrs, s)
torch.cuda.synchronize()
path = os.environ["LSB_GEMM_TRACE"]
native.setenv("LSB_GEMM_TRACE", path)
backend.run_device(k, ptrs, s)
torch.cuda.synchronize()
native.setenv("LSB_GEMM_TRACE", None)
rows = [[int(x) for x in line.split()] for line in open(path)]
ev = np.array(rows, dtype=np.float64)
base = ev[ev > 0].min()
ev = np.where(ev > 0, ev - base, np.nan)
print("ev3 milestones:", [int(x) for x in ev[3][:8] if not np.isnan(x)])
for u in range(4):
    seg = ev[3][8 + 8 * u:14 + 8 * u]
    if not np.isnan(seg[0]):
        print(f"unit round {u}: store start {int(seg[0])}, blocks", [int(x - seg[0]) for x in seg[1:5] if not np.isnan(x)],
              "end", int(seg[5] - seg[0]) if not np.isnan(seg[5]) else None)
print("ev2 MMA chunk starts:", [int(x) for x in ev[2][:20] if not np.isnan(x)])
print("ev1 epi chunk ready :", [int(x) for x in ev[1][:20] if not np.isnan(x)])
st = ev[0][:64]
d = np.diff(st[~np.isnan(st)])
print("ev0 stage intervals (last tile): median %.0f  p90 %.0f  max %.0f  (n=%d)" % (np.median(d), np.percentile(d, 90), d.max(), len(d)))
print("ev0:", [int(x) for x in st if not np.isnan(x)])
