"""Timeline of the blocked 3xTF32 execute (backend._execute_blocked) on C5:
when each piece upload, split, rectangle and download finishes, on the device
clock (timing events recorded on the backend's own streams after each op).

    python tools/blocked_timeline.py [--n 16384] [--pieces 8] [--reps 3]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_00618_b200 import backend, native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--n", type=int, default=0, help="resize C5's m = k = n")
ap.add_argument("--pieces", type=int, default=0, help="0: the backend rule")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
native.init(0)
backend.BLOCK_PIECES = args.pieces or None
n = args.n
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import common  # noqa: E402
from paper_2205_00618_b200 import shard  # noqa: E402
import json  # noqa: E402

gj = common.graph_json(common.config(args.config)["graph"])
if n:
    obj = json.loads(gj)
    for v in ("m", "k", "n"):
        obj = shard.shard_graph(obj, n, v)
    gj = json.dumps(obj)
k = backend.compile_graph(gj)
rng = np.random.default_rng(0)
bufs, pinned = {}, []
for s, shp in k.slot_shapes.items():
    pb = native.PinnedBuffer(tuple(shp))
    pinned.append(pb)          # the array does not own the allocation
    if s in k.input_slots:
        pb.array[:] = rng.uniform(-1, 1, size=shp).astype(np.float32)
    bufs[s] = pb.array

marks = []
t0 = [None]
real = {"h2d": native.h2d, "h2d_2d": native.h2d_2d, "d2h_2d": native.d2h_2d}


def mark(name, stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(torch.cuda.ExternalStream(stream))
    marks.append((name, e))


def wrap(name):
    def f(*a):
        real[name](*a)
        mark(name, a[-1])
    return f


native.h2d, native.h2d_2d, native.d2h_2d = wrap("h2d"), wrap("h2d_2d"), wrap("d2h_2d")
real_lb = backend.Runner.launch_blocked


def lb(self, slots, stream, flags, gen, r0, r1, c0, c1):
    n_ = real_lb(self, slots, stream, flags, gen, r0, r1, c0, c1)
    mark({2: "prepA", 4: "prepB", 8: "rect", 24: "grow"}.get(flags, str(flags)) + f"[{r0}:{r1},{c0}:{c1}]", stream)
    return n_


backend.Runner.launch_blocked = lb
for rep in range(args.reps + 1):
    marks.clear()
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    torch.cuda.synchronize()
    w = time.perf_counter()
    backend.execute(k, bufs)
    wall = (time.perf_counter() - w) * 1e3
    torch.cuda.synchronize()
    if rep == 0:
        continue
    print(f"rep {rep}: wall {wall:.2f} ms")
    if rep == args.reps:
        for name, e in marks:
            print(f"  {start.elapsed_time(e):8.2f}  {name}")
