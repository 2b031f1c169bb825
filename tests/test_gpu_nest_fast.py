"""The 32-bit row-walking and tiled-transpose nest kernels (csrc/nest_fast.cuh)
against the general affine_nest_kernel and the oracle.

Both families apply the reference's operations in the same order
(feedback.py:144-170), so a nest must give the same bytes through either; the
acceptance nests (maxpool, transpose, concat, broadcast_add --
op_graphs.py:27-36, 89-98) resized to ragged shapes are checked against the
oracle too, with the launched kernel asserted.
"""
from __future__ import annotations

import json

import numpy as np
import pytest

import common
from oracle import oracle as O
from paper_2205_00618_b200 import backend, native, shard

pytestmark = pytest.mark.gpu

IDX = common.index()


def _has_nest(case) -> bool:
    k = backend.compile_graph(common.graph_json(case["graph"]))
    return any(s.kind == "nest" for s in k.plan.steps)


NEST_CASES = [c for c in IDX["cases"] if _has_nest(c)]


def _run(gj, bufs):
    k = backend.compile_graph(gj)
    got = {s: np.array(b, copy=True) for s, b in bufs.items()}
    backend.execute(k, got)
    return k, got


def _same_bytes(a, b):
    return np.array_equal(np.ascontiguousarray(a, dtype=np.float32).view(np.uint32),
                          np.ascontiguousarray(b, dtype=np.float32).view(np.uint32))


@pytest.mark.parametrize("case", NEST_CASES, ids=[c["name"] for c in NEST_CASES])
def test_fast_nest_matches_general_kernel(case, monkeypatch):
    gj = common.graph_json(case["graph"])
    ins, ref, _ = common.case_data(case)
    _, fast = _run(gj, ins)
    monkeypatch.setenv("LSB_NO_NEST_FAST", "1")
    _, gen = _run(gj, ins)
    assert native.last_nest_kernel() == 0
    for slot in ref:
        assert _same_bytes(fast[slot], gen[slot]), f"{case['name']} slot {slot}"


def _graph(name, sizes):
    case = next(c for c in IDX["cases"] if c["name"] == name)
    g = json.loads(common.graph_json(case["graph"]))
    for var, n in sizes.items():
        g = shard.shard_graph(g, n, var)
    if name == "acc_concat":
        # the second operand's view starts where the first ends (the golden
        # graph's -3 is its own c1): keep the resized graph a concat
        for node in g["nodes"]:
            for c in node.get("constraints", []):
                if c["offset"] == -3:
                    c["offset"] = -sizes["c1"]
    return json.dumps(g)


RESIZED = [
    ("acc_maxpool", {"h": 260, "w": 1002, "r": 130, "c": 501}, 1),
    ("acc_maxpool", {"h": 64, "w": 12, "r": 32, "c": 6}, 1),
    ("acc_maxpool", {"h": 70, "w": 1000, "r": 35, "c": 500}, 4),
    ("acc_maxpool", {"h": 6, "w": 40, "r": 3, "c": 20}, 4),
    ("acc_transpose", {"a": 300, "b": 517, "r": 517, "c": 300}, 2),
    ("acc_transpose", {"a": 33, "b": 8, "r": 8, "c": 33}, None),
    ("acc_transpose", {"a": 300, "b": 516, "r": 516, "c": 300}, 5),
    ("acc_transpose", {"a": 64, "b": 128, "r": 128, "c": 64}, 5),
    ("acc_concat", {"r": 129, "c1": 200, "c2": 333, "c": 533}, 1),
    ("acc_concat", {"r": 129, "c1": 200, "c2": 332, "c": 532}, 3),
    ("acc_concat", {"r": 33, "c1": 202, "c2": 334, "c": 536}, None),
    ("acc_broadcast_add", {"m": 257, "n": 1030}, 1),
    ("acc_broadcast_add", {"m": 257, "n": 1032}, 3),
    ("acc_broadcast_add", {"m": 9, "n": 4096}, 3),
    ("acc_broadcast_add", {"m": 3000, "n": 5}, 1),
]


@pytest.mark.parametrize("name,sizes,kind", RESIZED, ids=[f"{n}-{i}" for i, (n, _, _) in enumerate(RESIZED)])
def test_resized_acceptance_nests(name, sizes, kind, monkeypatch):
    try:
        gj = _graph(name, sizes)
    except Exception as e:   # a size var this graph does not have
        pytest.skip(str(e))
    k = backend.compile_graph(gj)
    rng = np.random.default_rng(11)
    ins = {s: rng.integers(-50, 51, size=shp).astype(np.float32) for s, shp in k.slot_shapes.items()
           if s in k.input_slots}
    ref = O.reference_eval(gj, ins)
    _, fast = _run(gj, ins)
    got_kind = native.last_nest_kernel()
    if kind is not None:
        assert got_kind == kind, f"{name}: kernel {got_kind}"
    monkeypatch.setenv("LSB_NO_NEST_FAST", "1")
    _, gen = _run(gj, ins)
    for slot, r in ref.items():
        want = np.asarray(r, dtype=np.float64).astype(np.float32).reshape(fast[slot].shape)
        assert np.array_equal(fast[slot], want), f"{name} slot {slot} vs oracle"
        assert _same_bytes(fast[slot], gen[slot]), f"{name} slot {slot} vs general kernel"
