"""Row-sharded C5 computed shard by shard on the device.

The GPU box gives one GPU per call, so the P-rank job is run here as its P
shards one after another on cuda:0, each exactly as rank r of P runs it in
bench.py (the shard graph with the M var resized, that rank's rows of A, the
full B) and each checked on sampled rows against f64.  The assembled C is
then checked on rows drawn from every shard -- what the optional all-gather
delivers to every rank."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c5_inputs():
    rng = np.random.default_rng(4)
    A = rng.uniform(-1, 1, (16384, 16384)).astype(np.float32)
    B = rng.uniform(-1, 1, (16384, 16384)).astype(np.float32)
    return A, B


def _graph(rows):
    from paper_2205_00618_b200.shard import shard_graph
    with open(os.path.join(ROOT, "tests", "golden", "graphs", "C5.json")) as f:
        return shard_graph(json.load(f), rows)


def _metric(got, ref):
    d = (got - ref).abs()
    return float(d.max() / max(float(ref.abs().max()), 1.0)), float((d <= 1e-5 + 1e-4 * ref.abs()).double().mean())


@pytest.mark.parametrize("world", [2, 8])
def test_c5_row_shards_match_f64(c5_inputs, world):
    import torch
    from paper_2205_00618_b200 import backend, native
    from paper_2205_00618_b200.shard import shard_rows
    native.init(0)
    A, B = c5_inputs
    dev = torch.device("cuda", 0)
    Bd = torch.from_numpy(B).to(dev)
    B64 = Bd.double()
    C = torch.empty((16384, 16384), dtype=torch.float32, device=dev)
    for rank in range(world):
        r0, r1 = shard_rows(16384, world, rank)
        k = backend.compile_graph(_graph(r1 - r0))
        assert k.plan.steps[0].params["M"] == r1 - r0
        Ad = torch.from_numpy(A[r0:r1]).to(dev)
        Cs = C[r0:r1]
        n = backend.run_device(k, {0: Ad.data_ptr(), 1: Bd.data_ptr(), 2: Cs.data_ptr()},
                               torch.cuda.current_stream().cuda_stream)
        assert n >= 1
        torch.cuda.synchronize()
        idx = torch.tensor(sorted({0, (r1 - r0) // 2, r1 - r0 - 1, 127, 128}), device=dev)
        ref = Ad[idx].double() @ B64
        m, strict = _metric(Cs[idx].double(), ref)
        assert m <= 1e-4, (world, rank, m)
        # the VM itself fails the strict rule on ~0.6 % at K = 16384
        assert strict > 0.99, (world, rank, strict)
        del Ad
    # the assembled matrix: rows from every shard
    rows = sorted({int(x) for x in np.linspace(0, 16383, 3 * world)})
    Ad = torch.from_numpy(A[rows]).to(dev)
    m, strict = _metric(C[torch.tensor(rows, device=dev)].double(), Ad.double() @ B64)
    assert m <= 1e-4 and strict > 0.99, (m, strict)
