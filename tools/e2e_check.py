"""e2e check of row-streamed execute on C5-like shapes: correctness on sampled
rows + timing of execute() (pinned host buffers)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_00618_b200 import backend, native  # noqa: E402
from paper_2205_00618_b200.shard import shard_graph  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
gj = open("tests/golden/graphs/C5.json").read()
import json  # noqa: E402
obj = json.loads(gj)
for v in obj["vars"]:
    if v["origin"] is None:
        v["size"] = n
    else:
        v["size"] = v["origin"]["factor"] if v["origin"]["part"] == "inner" else -(-n // v["origin"]["factor"])
k = backend.compile_graph(obj)
rng = np.random.default_rng(0)
pa, pb, pc = native.PinnedBuffer((n, n)), native.PinnedBuffer((n, n)), native.PinnedBuffer((n, n))
pa.array[...] = rng.uniform(-1, 1, (n, n)).astype(np.float32)
pb.array[...] = rng.uniform(-1, 1, (n, n)).astype(np.float32)
bufs = {0: pa.array, 1: pb.array, 2: pc.array}
backend.execute(k, bufs)
ts = []
for _ in range(3):
    t = time.perf_counter()
    backend.execute(k, bufs)
    ts.append(time.perf_counter() - t)
rows = np.array([0, 1, n // 3, n - 1])
ref = pa.array[rows].astype(np.float64) @ pb.array.astype(np.float64)
err = np.max(np.abs(pc.array[rows] - ref) / np.maximum(np.abs(ref), 1))
print(f"n={n} streamed={backend._row_stream_plan(k, {0: 1}) is not None} e2e {min(ts)*1e3:.1f} ms "
      f"{2*n**3/min(ts)/1e12:.1f} TFLOP/s  launches {k.counters['launches']}  ref-metric {err:.2e}")
