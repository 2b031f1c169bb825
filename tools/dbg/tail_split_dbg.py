import json, os, sys
import numpy as np
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "tests")]
import common
from oracle import oracle as O
from paper_2205_00618_b200 import backend, shard
os.environ["LSB_GEMM_ALGO"] = "tf32x3"
m, k, n = 2048, 1024, 2560
case = next(c for c in common.index()["cases"] if c["name"] == "semiring_mul_add")
obj = json.loads(common.graph_json(case["graph"]))
for var, sz in dict(m=m, k=k, n=n).items():
    obj = shard.shard_graph(obj, sz, var)
gj = json.dumps(obj)
kern = backend.compile_graph(gj)
rng = np.random.default_rng(3)
A = rng.standard_normal((m, k)).astype(np.float32)
B = rng.standard_normal((k, n)).astype(np.float32)
for nonfin in (False, True):
    A2, B2 = A.copy(), B.copy()
    if nonfin:
        A2[m - 1, 3] = np.inf
        B2[1, n - 1] = np.nan
    for split in (True, False):
        if split: os.environ.pop("LSB_NO_TAIL_SPLIT", None)
        else: os.environ["LSB_NO_TAIL_SPLIT"] = "1"
        bufs = {0: A2.copy(), 1: B2.copy()}
        backend.execute(kern, bufs)
        C = bufs[2].reshape(m, n).astype(np.float64)
        ref = A2.astype(np.float64) @ B2.astype(np.float64)
        fin = np.isfinite(ref)
        d = np.where(fin, np.abs(C - ref), 0)
        bad = fin & ~(d <= 1e-5 + 1e-4 * np.abs(ref))
        print("nonfin", nonfin, "split", split, "bad", bad.sum(), "maxd", d.max(), "at", np.unravel_index(d.argmax(), d.shape),
              "bad rows", np.unique(np.argwhere(bad)[:, 0])[:10], "bad cols", np.unique(np.argwhere(bad)[:, 1])[:10])
