"""Seeded shape fuzz over every tuned and generic operator pair (reference
ir.py:178-222 OP_SEMANTICS), sized to reach each kernel path the dispatcher
picks -- one-launch small kernel, register-blocked SIMT (+ split-K), stream-K
fixup / cluster max-plus, 3xTF32 tensor cores, the generic-pair kernels --
against the f64 oracle on sampled output rows.  Small-integer inputs keep
every path exact (sums of products of integers < 2^24 are exact in fp32 and
in 3xTF32), so the comparison is bit-exact for every pair."""
import json

import numpy as np
import pytest

from oracle import oracle as O
from test_gpu_edges import _graph, _inputs, _run, _same

pytestmark = pytest.mark.gpu

PAIRS = ["mul_add", "add_max", "add_min", "mul_max", "mul_min", "add_add", "add_mul", "mul_mul"]
SIZES = [(1, 64), (60, 300), (250, 700), (900, 1600)]


def _cases(n=96, seed=2205):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        pair = PAIRS[i % len(PAIRS)]
        lo, hi = SIZES[(i // len(PAIRS)) % len(SIZES)]
        m, k, nn = (int(x) for x in rng.integers(lo, hi + 1, size=3))
        if pair in ("add_mul", "mul_mul"):
            k = min(k, 6)           # products of many integers overflow fp32 exactness
        out.append((pair, m, k, nn))
    return out


@pytest.mark.parametrize("pair,m,k,n", _cases(), ids=lambda v: str(v))
def test_fuzz_contraction(pair, m, k, n):
    gj = _graph(f"semiring_{pair}", m=m, k=k, n=n)
    lo, hi = (-2, 3) if pair in ("add_mul", "mul_mul") else (-4, 5)
    kern, ins = _inputs(gj, m * 7919 + k * 31 + n, lo, hi)
    got = _run(kern, ins)
    mvar = [v["id"] for v in json.loads(gj)["vars"] if v["name"] == "m"][0]
    rows = np.unique(np.array([0, m // 3, m // 2, m - 1]))
    ref = O.reference_eval(gj, ins, restrict={mvar: rows})
    out = next(iter(ref))
    _same(got[out].reshape(m, n)[rows], ref[out], exact=True)
