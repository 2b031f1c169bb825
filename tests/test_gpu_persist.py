"""Persistent 3xTF32 GEMM launch (TcArgs::units, the 128x256 tile geometry
when there are more units than SMs): ragged edges, the K-half tail split
(units = whole tiles + split halves walked by 148 CTAs) and the bias+ReLU fast
epilogue stored from registers, against the f64 oracle (integer inputs keep
3xTF32 exact) and bit-for-bit against the one-unit-per-CTA launch."""
import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_2205_00618_b200 import native
from test_gpu_edges import _graph, _inputs, _run, _same

pytestmark = pytest.mark.gpu

# (m, k, n): 4096x4096 = 512 tiles -> 444 whole + 68 split tiles (C4's layout);
# ragged m/n with partial last tiles and an even m-tile count (the 2-CTA
# cluster path: 16 x 17 = 272 tiles); 17 x 12 tiles, odd m-tiles (no pairs);
# one K chunk (no split: chunks < 2).  Every shape has more tiles than SMs,
# so the persistent instance runs (asserted through lsb_last_gemm_launch).
SHAPES = [(4096, 200, 4096), (2000, 300, 4100), (2050, 70, 3000), (1536, 64, 6144)]


@pytest.mark.parametrize("m,k,n", SHAPES, ids=lambda v: str(v))
def test_persistent_gemm_matches_oracle_and_single_unit(m, k, n, monkeypatch):
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    monkeypatch.setenv("LSB_TC_CFG", "16x256")
    gj = _graph("semiring_mul_add", m=m, k=k, n=n)
    kern, ins = _inputs(gj, m * 131 + k * 7 + n)
    got = _run(kern, ins)
    launch = native.last_gemm_launch()
    assert launch["bn"] == 256 and launch["units"] > launch["ctas"] > 0, launch
    assert launch["pair"] == (1 if -(-m // 128) % 2 == 0 else 0), launch
    out = next(s for s in got if s not in ins)
    mvar = [v["id"] for v in json.loads(gj)["vars"] if v["name"] == "m"][0]
    rows = np.unique(np.array([0, 127, 128, m // 2, m - 129, m - 1]).clip(0, m - 1))
    ref = O.reference_eval(gj, ins, restrict={mvar: rows})
    _same(got[out].reshape(m, n)[rows], ref[next(iter(ref))], exact=True)
    monkeypatch.setenv("LSB_NO_PERSIST", "1")
    single = _run(kern, ins)
    assert native.last_gemm_launch()["units"] == 0
    assert np.array_equal(got[out].view(np.uint32), single[out].view(np.uint32))


def test_persistent_fused_bias_relu(monkeypatch):
    """The bias + ReLU pipeline (C4's, fused into the epilogue) at C4's tile
    count through the persistent register store: exact against the oracle and
    bit-for-bit equal to the staged single-unit store."""
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    monkeypatch.setenv("LSB_TC_CFG", "16x256")
    import os
    m, n = 4096, 4096
    with open(os.path.join(os.path.dirname(__file__), "golden", "graphs", "C4.json")) as f:
        gj = f.read()
    kern, ins = _inputs(gj, 44)
    got = _run(kern, ins)
    rows = np.array([0, 1, 129, 2047, 4095])
    out = [s for s in got if s not in ins][-1]
    x, w, b = (ins[s] for s in sorted(ins))
    ref = np.maximum(x[rows].astype(np.float64) @ w.astype(np.float64) + b.reshape(1, -1), 0.0)
    _same(got[out].reshape(m, n)[rows], ref, exact=True)
    monkeypatch.setenv("LSB_NO_PERSIST", "1")
    single = _run(kern, ins)
    assert np.array_equal(got[out].view(np.uint32), single[out].view(np.uint32))
