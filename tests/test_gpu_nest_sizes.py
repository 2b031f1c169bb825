"""The affine-nest coverage kernel (affine_nest.cuh) on the reference's
acceptance nests resized to long, ragged rows (the golden ones are a few
points wide), against the oracle's reference_eval: exact (max, copies and
single adds of small integers), guards (maxpool windows, concat halves)
included."""

import numpy as np
import pytest

from oracle import oracle as O
from test_gpu_edges import _graph, _inputs, _run, _same

pytestmark = pytest.mark.gpu

CASES = [
    ("acc_maxpool", dict(h=82, w=80, r=41, c=40)),
    ("acc_maxpool", dict(h=70, w=130, r=35, c=65)),
    ("acc_transpose", dict(a=70, b=45, r=45, c=70)),
    ("acc_transpose", dict(a=333, b=33, r=33, c=333)),
    ("acc_concat", dict(r=33, c1=40, c2=27, c=67)),
    ("acc_broadcast_add", dict(m=50, n=77)),
    ("acc_broadcast_add", dict(m=3, n=1000)),
]


@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{'x'.join(map(str, s.values()))}" for n, s in CASES])
def test_nest_resized(name, sizes):
    gj = _graph(name, **sizes)
    kern, ins = _inputs(gj, 7)
    assert [s.kind for s in kern.plan.steps] == ["nest"]
    got = _run(kern, ins)
    ref = O.reference_eval(gj, ins)
    for s in ref:
        _same(got[s], ref[s], exact=True)
