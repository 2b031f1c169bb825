"""Schedules -> launch configurations, measured.

Builds contractions with the reference frontend (baseline/_ref, or
/root/reference/pkg/src here), compiles each schedule with the B200 backend
and times run_device on resident buffers (CUDA graph of the plan, L2 flushed
between steps, CUDA events).  Prints one JSON line per (shape, schedule):
the tiles the schedule selected, the modeled memory accesses the tuner ranks
by, and the measured time.

    python tools/schedule_sweep.py > profiles/r02_schedule_sweep.jsonl
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src", ROOT):
    if os.path.isdir(p) and p not in sys.path:
        sys.path.insert(0, p)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import loopsmith as ls  # noqa: E402
import torch  # noqa: E402
from loopsmith import schedule as sch  # noqa: E402

from paper_2205_00618_b200 import backend, native  # noqa: E402


def reorder(g, order):
    for node in g:
        names = [v.name for v in node.order]
        sch.apply_action(g, sch.ReorderAction(node.id, [n for n in order if n in names]
                                              + [n for n in names if n not in order]))


def semiring(m, k, n, pair):
    b = ls.GraphBuilder()
    vm, vk, vn = b.var("m", m), b.var("k", k), b.var("n", n)
    a, bb = b.input("a", [vm, vk]), b.input("b", [vk, vn])
    rhs = a[vm, vk] + bb[vk, vn] if pair == ("max", "add") else a[vm, vk] * bb[vk, vn]
    c = b.contract("c", (vm, vn), rhs, op_pair=pair)
    b.output(c)
    return b.build()


SCHEDULES = {
    "naive": ([], None),
    "row n16": ([("n", 16)], ["m", "n_o", "k", "n_i"]),
    "block 4x64": ([("m", 4), ("n", 64)], ["m_o", "n_o", "k", "m_i", "n_i"]),
    "k-outer x8, block 4x64": ([("k", None), ("m", 4), ("n", 64)], ["k_o", "m_o", "n_o", "k_i", "m_i", "n_i"]),
}


def build(shape, pair, name):
    m, k, n = shape
    g = semiring(m, k, n, pair)
    splits, order = SCHEDULES[name]
    for var, f in splits:
        sch.split(g, sch.find_var(g, var), f if f is not None else k // 8)
    if order:
        reorder(g, order)
    return backend.compile_tree(ls.lower(g), ls.avx512_like())


def time_kernel(k, steps=20):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    t = {s: (torch.from_numpy(rng.uniform(-1, 1, shp).astype(np.float32)).to(dev) if s in k.input_slots
             else torch.zeros(shp, device=dev)) for s, shp in k.slot_shapes.items()}
    ptrs = {s: x.data_ptr() for s, x in t.items()}
    stream = torch.cuda.current_stream()
    for _ in range(3):
        backend.run_device(k, ptrs, stream.cuda_stream)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        backend.run_device(k, ptrs, torch.cuda.current_stream().cuda_stream)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        graph.replay()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    native.init(0)
    for shape, pair in (((4096, 1024, 4096), ("add", "mul")), ((2048, 2048, 2048), ("add", "mul")),
                        ((1024, 1024, 1024), ("max", "add")), ((256, 4096, 256), ("add", "mul"))):
        for name in SCHEDULES:
            k = build(shape, pair, name)
            st = next(s for s in k.plan.steps if s.kind == "gemm")
            ms = time_kernel(k)
            k._count(1)
            p = st.params
            flops = 2 * shape[0] * shape[1] * shape[2]
            print(json.dumps({"shape": list(shape), "pair": list(pair), "schedule": name,
                              "selected": {"algo": p.get("algo_selected"), "tile_m": p["tile_m"],
                                           "tile_n": p["tile_n"], "split_k": p["split_k"],
                                           "block": [p["schedule"].m_block, p["schedule"].n_block]},
                              "modeled_mem_accesses": k.memory_access_count(),
                              "ms": round(ms, 4), "TFLOP/s": round(flops / (ms * 1e-3) / 1e12, 2)}), flush=True)


if __name__ == "__main__":
    main()
