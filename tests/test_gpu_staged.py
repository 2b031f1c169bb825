"""Ordinary (pageable) host buffers through `execute`: copies larger than
backend.STAGE_MIN_BYTES cross PCIe through liblsb's pinned staging slots
(lsb_stage_*), in every execute schedule -- plain, row-streamed and blocked
(A row pieces, pitched B column pieces, pitched output rectangles).  Results
must equal the same call from page-locked buffers byte for byte."""
import json

import numpy as np
import pytest

import common
from paper_2205_00618_b200 import backend, native, shard

pytestmark = pytest.mark.gpu


def _graph(name, **sizes):
    case = next(c for c in common.index()["cases"] if c["name"] == name)
    obj = json.loads(common.graph_json(case["graph"]))
    for var, n in sizes.items():
        obj = shard.shard_graph(obj, n, var)
    return json.dumps(obj)


def _pinned_copy(a):
    pb = native.PinnedBuffer(a.shape)
    pb.array[...] = a
    return pb


def _both(k, ins):
    assert not any(native.is_pinned(a.ctypes.data) for a in ins.values())
    pageable = {s: a.copy() for s, a in ins.items()}
    backend.execute(k, pageable)
    keep = {s: _pinned_copy(a) for s, a in ins.items()}
    outs = {s: native.PinnedBuffer(k.slot_shapes[s]) for s in k.output_slots}
    pinned = {s: pb.array for s, pb in keep.items()}
    pinned.update({s: pb.array for s, pb in outs.items()})
    assert all(native.is_pinned(a.ctypes.data) for a in pinned.values())
    backend.execute(k, pinned)
    for s in k.output_slots:
        a = pageable[s].reshape(-1)
        b = np.array(pinned[s]).reshape(-1)
        assert np.array_equal(a, b), f"slot {s}: staged result differs"
    return pageable


@pytest.mark.parametrize("m,k,n", [(1536, 700, 2304), (2048, 512, 1536)])
def test_blocked_schedule_from_pageable(m, k, n, monkeypatch):
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    monkeypatch.setattr(backend, "STREAM_MIN_MACS", 0)
    kern = backend.compile_graph(_graph("semiring_mul_add", m=m, k=k, n=n))
    rng = np.random.default_rng(5)
    ins = {s: rng.integers(-4, 5, size=shp).astype(np.float32) for s, shp in kern.slot_shapes.items()
           if s in kern.input_slots}
    out = _both(kern, ins)
    (oslot,) = kern.output_slots
    want = ins[0].astype(np.float64).reshape(m, k) @ ins[1].astype(np.float64).reshape(k, n)
    assert np.array_equal(out[oslot].reshape(m, n), want.astype(np.float32))


def test_plain_schedule_from_pageable_conv():
    cfg = common.config("C3")
    kern = backend.compile_graph(common.graph_json(cfg["graph_guarded"]))
    ins = common.config_inputs("C3g")
    _both(kern, ins)


def test_staged_2d_pitched_roundtrip():
    """lsb_stage_h2d_2d / d2h_2d with pitches != widths (rows wider than a
    staging slot and narrow ones) move exactly the rectangle."""
    import torch
    native.init(0)
    rows, cols = 300, 5000
    host = np.random.default_rng(1).standard_normal((rows, cols)).astype(np.float32)
    dev = torch.zeros((rows, cols + 16), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    native.stage_h2d_2d(dev.data_ptr() + 4 * 3, 4 * (cols + 16), host.ctypes.data, 4 * cols, 4 * (cols - 7), rows, s)
    back = np.zeros((rows, cols), np.float32)
    native.stage_d2h_2d(back.ctypes.data, 4 * cols, dev.data_ptr() + 4 * 3, 4 * (cols + 16), 4 * (cols - 7), rows, s)
    torch.cuda.synchronize()
    native.stage_wait()
    assert np.array_equal(back[:, :cols - 7], host[:, :cols - 7]) and not back[:, cols - 7:].any()
    big = np.random.default_rng(2).standard_normal(40 << 20 >> 2).astype(np.float32)   # 40 MB, > 2 slots
    d = torch.empty(big.size, dtype=torch.float32, device="cuda")
    native.stage_h2d_2d(d.data_ptr(), big.nbytes, big.ctypes.data, big.nbytes, big.nbytes, 1, s)
    out = np.empty_like(big)
    native.stage_d2h_2d(out.ctypes.data, big.nbytes, d.data_ptr(), big.nbytes, big.nbytes, 1, s)
    torch.cuda.synchronize()
    native.stage_wait()
    assert np.array_equal(out, big)
