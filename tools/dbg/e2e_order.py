"""C5 execute() from pinned host buffers: the blocked schedule's B pieces
(default: as many as A's) against B whole first (one column piece)."""
import os, sys
import numpy as np
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2205_00618_b200 import backend, native
native.init(0)
cfg = os.environ.get("CFG", "C5")
k = backend.compile_graph(bench.load_graph(cfg))
host = bench.make_inputs(cfg)
keep, bufs = [], {}
for s_, shp in k.slot_shapes.items():
    pbuf = native.PinnedBuffer(tuple(shp))
    keep.append(pbuf)
    if s_ in host:
        pbuf.array[...] = host[s_].reshape(shp)
    bufs[s_] = pbuf.array
flops = k.flops
real = backend._blocked_plan
for mode in sys.argv[1:] or ["pieces", "bwhole"]:
    npieces = int(mode.split(":")[1]) if ":" in mode else None
    backend.BLOCK_PIECES = npieces
    def plan(*a, _m=mode):
        bp = real(*a)
        if bp is not None and _m.startswith("bwhole"):
            bp["cols"] = [(0, bp["N"])]
        return bp
    backend._blocked_plan = plan
    backend.execute(k, bufs)
    ts = []
    for _ in range(9):
        t0 = time.perf_counter(); backend.execute(k, bufs); ts.append(time.perf_counter() - t0)
    print(mode, ": %.1f ms median, %.1f TF/s" % (np.median(ts) * 1e3, flops / np.median(ts) / 1e12), flush=True)
