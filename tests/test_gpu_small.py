"""Latency-bound contractions on the one-launch small kernel
(csrc/small_gemm.cuh): parity with the oracle on ragged tiles and ragged
K chunks, every tuned operator pair, non-finite tropical inputs, and the
launch count that shows the kernel ran alone (no split-K fold)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2205_00618_b200 import native
from test_gpu_edges import _graph, _inputs, _run, _same

pytestmark = pytest.mark.gpu

SHAPES = [(4, 4, 4), (33, 100, 36), (256, 256, 256), (64, 1024, 64), (300, 132, 200), (31, 4, 1000)]


@pytest.mark.parametrize("case", ["semiring_mul_add", "semiring_add_max", "semiring_add_min"])
@pytest.mark.parametrize("shape", SHAPES)
def test_small_kernel_parity(case, shape):
    m, k, n = shape
    gj = _graph(case, m=m, k=k, n=n)
    kern, ins = _inputs(gj, 23)
    n0 = native.launch_count()
    got = _run(kern, ins)
    assert native.launch_count() - n0 == 1, "small sizes run as one launch"
    ref = O.reference_eval(gj, ins)
    out = next(iter(ref))
    _same(got[out], ref[out], exact=True)   # small integers: exact for sums too


@pytest.mark.parametrize("shape", [(33, 100, 36), (128, 512, 64)])
def test_small_kernel_uniform_sum_tolerance(shape):
    m, k, n = shape
    gj = _graph("semiring_mul_add", m=m, k=k, n=n)
    kern, _ = _inputs(gj, 0)
    rng = np.random.default_rng(5)
    ins = {s: rng.uniform(-1, 1, size=shp).astype(np.float32)
           for s, shp in kern.slot_shapes.items() if s in kern.input_slots}
    got = _run(kern, ins)
    ref = O.reference_eval(gj, ins)
    out = next(iter(ref))
    _same(got[out], ref[out], exact=False)


@pytest.mark.parametrize("op", ["semiring_add_max", "semiring_add_min"])
def test_small_kernel_tropical_nonfinite(op):
    gj = _graph(op, m=40, k=68, n=24)
    kern, ins = _inputs(gj, 29)
    rng = np.random.default_rng(3)
    for a in ins.values():
        flat = a.reshape(-1)
        idx = rng.choice(flat.size, size=12, replace=False)
        flat[idx[:4]] = np.inf
        flat[idx[4:8]] = -np.inf
        flat[idx[8:]] = np.nan
    got = _run(kern, ins)
    ref = O.reference_eval(gj, ins)
    out = next(iter(ref))
    _same(got[out], ref[out], exact=True)


def test_small_kernel_fused_epilogue_and_batch():
    import common
    for name in ("mlp_bias_relu_small", "batched_gemm"):
        c = next(x for x in common.index()["cases"] if x["name"] == name)
        gj = common.graph_json(c["graph"])
        ins, _, _ = common.case_data(c)
        from paper_2205_00618_b200 import backend
        kern = backend.compile_graph(gj)
        got = _run(kern, ins)
        ref = O.reference_eval(gj, ins)
        for slot, r in ref.items():
            ok, msg = common.check_case(c["rule"], got[slot].reshape(r.shape), r)
            assert ok, f"{name}: {msg}"
