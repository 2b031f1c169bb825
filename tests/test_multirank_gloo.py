"""Row-sharded multi-rank path on CPU (world_size 2, gloo).

The GPU box offers one GPU per call, so the N>1 host logic -- shard
boundaries, the resized shard graph, the planner on it, the rank's seeded
input slice and the optional all-gather of C -- runs here in two processes,
with the oracle standing in for each rank's kernel."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import common
from paper_2205_00618_b200.shard import shard_graph, shard_rows


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, graph, A, B, q):
    import torch
    from oracle import oracle as O
    from paper_2205_00618_b200.graph import Graph
    from paper_2205_00618_b200.planner import plan_graph
    from paper_2205_00618_b200.shard import gather_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, r1 = shard_rows(A.shape[0], world, rank)
        g = shard_graph(graph, r1 - r0)
        plan = plan_graph(g)
        step = plan.steps[0]
        assert step.kind == "gemm" and step.params["M"] == r1 - r0
        out = O.reference_eval(Graph.from_json(g), {0: A[r0:r1], 1: B})[2]
        full = gather_rows(torch.from_numpy(out.astype(np.float32)), world)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [64, 37])
def test_two_rank_row_shards_gather_to_full_result(m):
    case = next(c for c in common.index()["cases"] if c["name"] == "semiring_add_max")
    graph = shard_graph(common.graph_json(case["graph"]), m)
    rng = np.random.default_rng(5)
    A = rng.uniform(-10, 10, (m, 29)).astype(np.float32)
    B = rng.uniform(-10, 10, (29, 53)).astype(np.float32)
    want = (A[:, :, None] + B[None, :, :]).max(axis=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, graph, A, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert np.array_equal(res[r], want.astype(np.float32))


def test_shard_rows_balanced():
    assert [shard_rows(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert [shard_rows(16384, 8, r)[1] - shard_rows(16384, 8, r)[0] for r in range(8)] == [2048] * 8
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)


def test_shard_graph_resizes_split_lineage():
    g = shard_graph(common.graph_json("graphs/C5.json"), 2048)
    sizes = {v["name"]: v["size"] for v in g["vars"]}
    assert sizes["m"] == 2048 and sizes["m_i"] == 4 and sizes["m_o"] == 512
    from paper_2205_00618_b200.planner import plan_graph
    assert plan_graph(g).steps[0].params["M"] == 2048
