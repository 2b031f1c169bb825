"""The blocked 3xTF32 schedule of `execute` (backend._execute_blocked): A row
pieces and B column pieces split into the resident workspace as they land
(LSB_GEMM_PREP_A / PREP_B), output rectangles computed from what is split
(LSB_GEMM_PRESPLIT) and copied back as pitched rectangles -- interleaved
(A0 B0 A1 B1 ...) or, for long reductions, B whole first and full row
strips per A piece (BLOCK_B_FIRST_K, forced here with b_first).

The schedule normally starts at 2^34 multiply-adds (C4, C5); here the
threshold is lowered so ragged mid-size problems take it, and each result is
checked against the oracle (reference_eval restatement) and against the
unblocked path.  Non-finite inputs exercise the per-sequence flags: a flagged
A row piece arrives after earlier rectangles already ran."""
import json

import numpy as np
import pytest

import common
from oracle import oracle as O
from paper_2205_00618_b200 import backend, native, shard

pytestmark = pytest.mark.gpu


def _graph(name, **sizes):
    case = next(c for c in common.index()["cases"] if c["name"] == name)
    obj = json.loads(common.graph_json(case["graph"]))
    for var, n in sizes.items():
        obj = shard.shard_graph(obj, n, var)
    return json.dumps(obj)


def _inputs(k, seed, normal=False):
    """Small integers (every summation order exact, so results compare
    exactly) or standard normals (nonzero lo parts; compared by the
    reference's metric and bitwise against the unblocked launch)."""
    rng = np.random.default_rng(seed)
    return {s: (rng.standard_normal(size=shp) if normal else rng.integers(-4, 5, size=shp)).astype(np.float32)
            for s, shp in k.slot_shapes.items() if s in k.input_slots}


def _blocked(monkeypatch):
    # (auto-selection keeps problems this small on the SIMT kernels)
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    monkeypatch.setattr(backend, "STREAM_MIN_MACS", 0)
    calls = []
    real = backend._execute_blocked

    def spy(*a, **kw):
        calls.append(a[-1])
        return real(*a, **kw)
    monkeypatch.setattr(backend, "_execute_blocked", spy)
    return calls


def _check(got, ref, exact=True):
    ref = np.asarray(ref, np.float64)
    got = np.asarray(got, np.float64).reshape(ref.shape)
    assert np.array_equal(np.isnan(ref), np.isnan(got)), "NaN mask differs"
    inf = np.isinf(ref)
    assert np.array_equal(got[inf], ref[inf])
    fin = np.isfinite(ref)
    if exact:
        assert np.array_equal(got[fin], ref[fin].astype(np.float32)), "finite values differ"
    else:
        assert common.ref_metric(got[fin], ref[fin]) <= 1e-4


@pytest.mark.parametrize("b_first", [False, True], ids=["interleaved", "b_first"])
@pytest.mark.parametrize("normal", [False, True], ids=["int", "normal"])
@pytest.mark.parametrize("shape", [(1000, 300, 1300), (512, 77, 512), (2304, 129, 700), (700, 1000, 2600)])
def test_blocked_mul_add(shape, normal, b_first, monkeypatch):
    calls = _blocked(monkeypatch)
    monkeypatch.setattr(backend, "BLOCK_B_FIRST_K", 0 if b_first else 1 << 40)
    m, kk, n = shape
    gj = _graph("semiring_mul_add", m=m, k=kk, n=n)
    k = backend.compile_graph(gj)
    ins = _inputs(k, 31, normal)
    bufs = {s: a.copy() for s, a in ins.items()}
    backend.execute(k, bufs)
    assert len(calls) == 1, "blocked schedule not taken"
    bp = calls[0]
    assert len(bp["rows"]) > 1 and (len(bp["cols"]) == 1 if b_first else len(bp["cols"]) > 1)
    ref = O.reference_eval(gj, ins)
    out, = ref
    _check(bufs[out], ref[out], exact=not normal)
    # and the same bytes as the unblocked 3xTF32 launch
    monkeypatch.setenv("LSB_NO_BLOCKED", "1")
    plain = {s: a.copy() for s, a in ins.items()}
    backend.execute(k, plain)
    assert np.array_equal(np.asarray(plain[out]).reshape(-1), np.asarray(bufs[out]).reshape(-1))


def test_blocked_bias_relu_epilogue(monkeypatch):
    calls = _blocked(monkeypatch)
    gj = _graph("mlp_bias_relu_small", b=1536, k=200, n=1100)
    k = backend.compile_graph(gj)
    ins = _inputs(k, 5, normal=True)
    bufs = {s: a.copy() for s, a in ins.items()}
    backend.execute(k, bufs)
    assert calls
    ref = O.reference_eval(gj, ins)
    for s in ref:
        _check(bufs[s], ref[s], exact=False)


@pytest.mark.parametrize("b_first", [False, True], ids=["interleaved", "b_first"])
def test_blocked_nonfinite_late_pieces(b_first, monkeypatch):
    """inf/NaN in the last A row piece and a middle B column piece: only the
    rectangles computed after those pieces land see the flags."""
    calls = _blocked(monkeypatch)
    monkeypatch.setattr(backend, "BLOCK_B_FIRST_K", 0 if b_first else 1 << 40)
    m, kk, n = 1280, 96, 1536
    gj = _graph("semiring_mul_add", m=m, k=kk, n=n)
    k = backend.compile_graph(gj)
    ins = _inputs(k, 9)
    A, B = ins[0], ins[1]
    A[m - 3, 7] = np.inf
    A[1100, 2] = np.nan
    B[5, 800] = -np.inf
    A[10, 5] = np.inf        # first piece too
    bufs = {s: a.copy() for s, a in ins.items()}
    backend.execute(k, bufs)
    assert calls
    ref = O.reference_eval(gj, ins)
    out, = ref
    _check(bufs[out], ref[out])
    # a clean second call reuses the workspace; stale flags must not leak
    clean = _inputs(k, 10)
    bufs = {s: a.copy() for s, a in clean.items()}
    backend.execute(k, bufs)
    ref = O.reference_eval(gj, clean)
    _check(bufs[out], ref[out])


def test_blocked_rejects_misaligned_rectangle():
    """PRESPLIT rectangles must lie on output-tile corners (lsb.h)."""
    gj = _graph("semiring_mul_add", m=512, k=64, n=512)
    k = backend.compile_graph(gj)
    ins = _inputs(k, 1)
    r = k.runner
    dev = r.slot_buffers()
    for s, a in ins.items():
        native.h2d(dev[s], a.ctypes.data, a.nbytes, 0)
    r.launch_blocked(dev, 0, native.GEMM_PREP_A | native.GEMM_PREP_B, 77, 0, 512, 0, 512)
    with pytest.raises(Exception, match="tile corners"):
        r.launch_blocked(dev, 0, native.GEMM_PRESPLIT, 77, 64, 512, 0, 512)
    with pytest.raises(Exception, match="nonzero gen"):
        r.launch_blocked(dev, 0, native.GEMM_PRESPLIT, 0, 0, 512, 0, 512)
    native.sync(0)
