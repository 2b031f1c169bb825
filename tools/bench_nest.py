"""The affine-nest coverage kernel (csrc/affine_nest.cuh) on realistic sizes:
the reference's ACCEPTANCE_OPS nests (maxpool, transpose, concat,
broadcast_add) resized, inputs resident in HBM, L2 flushed between calls;
achieved GB/s (algorithmic bytes: inputs read once + outputs written once)
against the measured HBM copy bandwidth.  python tools/bench_nest.py"""
import json
import os
import sys

import numpy as np
import torch

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [R, os.path.join(R, "tests")]
import common  # noqa: E402
from paper_2205_00618_b200 import backend, native, shard  # noqa: E402

CASES = {
    "acc_maxpool": {"h": 8192, "w": 8192, "r": 4096, "c": 4096},
    "acc_transpose": {"a": 8192, "b": 8192, "r": 8192, "c": 8192},
    "acc_concat": {"r": 8192, "c1": 4096, "c2": 4096, "c": 8192},
    "acc_broadcast_add": {"m": 8192, "n": 8192},
}


def graph(name, sizes):
    case = next(c for c in common.index()["cases"] if c["name"] == name)
    g = json.loads(common.graph_json(case["graph"]))
    for var, n in sizes.items():
        g = shard.shard_graph(g, n, var)
    if name == "acc_concat":   # the second view starts where the first ends (the golden graph's -3 is its c1)
        for node in g["nodes"]:
            for c in node.get("constraints", []):
                if c["offset"] == -3:
                    c["offset"] = -sizes["c1"]
    return json.dumps(g)


def main():
    native.init(0)
    try:
        peak = json.load(open(os.path.join(R, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        peak = None
    st = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    out = {}
    for name, sizes in CASES.items():
        k = backend.compile_graph(graph(name, sizes))
        t = {s: torch.rand(shp, device="cuda") for s, shp in k.slot_shapes.items()}
        ptrs = {s: v.data_ptr() for s, v in t.items()}
        nbytes = sum(4 * int(np.prod(shp)) for shp in k.slot_shapes.values())
        for _ in range(3):
            backend.run_device(k, ptrs, st.cuda_stream)
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            backend.run_device(k, ptrs, st.cuda_stream)
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ts]))
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"sizes": sizes, "kernels": [s.kind for s in k.plan.steps], "ms": round(ms, 4),
                     "bytes": nbytes, "GB/s": round(gbs, 1), "hbm_peak_GB/s": peak,
                     "frac_hbm": round(gbs / peak, 3) if peak else None}
        print(name, out[name], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
