"""Random affine nests through the C ABI (lsb_affine_nest): the fast kernels
(csrc/nest_fast.cuh) against the general affine_nest_kernel, bit for bit, and
both against a numpy restatement of the nest's meaning (feedback.py:144-170:
combine over the operands left to right, beta, reduce in loop order; guarded
reads take the fill, ir.py:238-245).

Operands are views into random buffers with random (also negative and zero)
coefficients, so strided, reversed, broadcast and transposed accesses, windows
with guards and 1-3 reduction dims all occur; small-integer data keeps every
summation order exact.
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest
import torch

from paper_2205_00618_b200 import native

pytestmark = pytest.mark.gpu

OPS = {0: lambda a, b: a + b, 1: lambda a, b: a * b, 2: np.maximum, 3: np.minimum}
IDENT = {0: 0.0, 1: 1.0, 2: -np.inf, 3: np.inf}


def _affine_vals(base, coeff, grids):
    v = np.full(grids[0].shape, base, dtype=np.int64)
    for c, g in zip(coeff, grids):
        v = v + c * g
    return v


def _random_nest(rng, aligned):
    n_out = int(rng.integers(1, 5))
    n_red = int(rng.integers(0, 4))
    q = 4 if aligned else 1
    ext_out = [int(rng.integers(1, 7)) for _ in range(n_out)]
    ext_out[-1] = int(rng.integers(1, 9)) * q if aligned else int(rng.integers(1, 40))
    ext_red = [int(rng.integers(1, 4)) for _ in range(n_red)]
    ext = ext_out + ext_red
    n_ops = int(rng.integers(1, 3))
    grids = np.meshgrid(*[np.arange(e) for e in ext], indexing="ij") if ext else []
    ops = []
    for _ in range(n_ops):
        coeff = [int(rng.integers(-2, 4)) * (q if i < len(ext) - 1 or not aligned else 1) for i in range(len(ext))]
        if aligned:   # innermost output dim contiguous or broadcast, other offsets whole float4s
            coeff = [c * 1 for c in coeff]
            coeff[n_out - 1] = int(rng.integers(0, 2))
        vals = _affine_vals(0, coeff, grids)
        base = int(-vals.min())
        if aligned:
            base = (base + 3) // 4 * 4
        size = int(vals.max() + base + 1)
        guards = []
        for _g in range(int(rng.integers(0, 3))):
            gco = [int(rng.integers(-1, 2)) for _ in ext]
            gv = _affine_vals(0, gco, grids)
            gbase = int(rng.integers(-2, 3))
            gsize = max(1, int(gv.max() - gv.min()) + int(rng.integers(-2, 3)))
            guards.append((gbase - int(gv.min()) - int(rng.integers(0, 2)), gco, gsize))
        ops.append({"base": base, "coeff": coeff, "size": size + (4 if aligned else 0), "guards": guards,
                    "fill": float(rng.integers(-3, 4))})
    # output: a permutation of a dense row-major layout (every point its own address)
    perm = list(rng.permutation(n_out)) if not aligned else list(range(n_out))
    strides = [0] * n_out
    acc = 1
    for d in reversed(perm):
        strides[d] = acc
        acc *= ext_out[d]
    return {"n_out": n_out, "n_red": n_red, "ext": ext, "ops": ops, "out_coeff": strides, "out_size": acc,
            # reduce: add / max / min (a long product of integers leaves f32's exact range)
            "combine": int(rng.integers(0, 4)), "reduce": int(rng.choice([0, 2, 3])),
            "beta": float(rng.choice([1.0, 1.0, 0.5, -2.0]))}


def _numpy_eval(nest, bufs):
    ext, n_out = nest["ext"], nest["n_out"]
    grids = np.meshgrid(*[np.arange(e) for e in ext], indexing="ij")
    t = None
    for op, buf in zip(nest["ops"], bufs):
        addr = _affine_vals(op["base"], op["coeff"], grids)
        ok = np.ones(addr.shape, bool)
        for gb, gco, gs in op["guards"]:
            gv = _affine_vals(gb, gco, grids)
            ok &= (gv >= 0) & (gv < gs)
        v = np.where(ok, buf[np.where(ok, addr, 0)], np.float32(op["fill"])).astype(np.float32)
        t = v if t is None else OPS[nest["combine"]](t, v).astype(np.float32)
    if nest["beta"] != 1.0:
        t = (np.float32(nest["beta"]) * t).astype(np.float32)
    if nest["n_red"]:
        red = tuple(range(n_out, len(ext)))
        r = nest["reduce"]
        # small integers (and halves / doubles of them): every order is exact
        t = {0: np.sum, 1: np.prod, 2: np.max, 3: np.min}[r](t.astype(np.float64), axis=red).astype(np.float32)
    out = np.zeros(nest["out_size"], np.float32)
    og = np.meshgrid(*[np.arange(e) for e in ext[:n_out]], indexing="ij")
    out[_affine_vals(0, nest["out_coeff"], og)] = t
    return out


def _run(nest, dev_bufs, out):
    d = native.NestDesc()
    d.n_out, d.n_red = nest["n_out"], nest["n_red"]
    for i, e in enumerate(nest["ext"]):
        d.extent[i] = e
    d.n_operands = len(nest["ops"])
    for o, (op, buf) in enumerate(zip(nest["ops"], dev_bufs)):
        no = d.operand[o]
        no.ptr = buf.data_ptr()
        no.addr.base = op["base"]
        for i, c in enumerate(op["coeff"]):
            no.addr.coeff[i] = c
        no.n_guards = len(op["guards"])
        for q, (gb, gco, gs) in enumerate(op["guards"]):
            no.guard[q].base = gb
            for i, c in enumerate(gco):
                no.guard[q].coeff[i] = c
            no.guard_size[q] = gs
        no.fill = op["fill"]
    d.out = out.data_ptr()
    for i, c in enumerate(nest["out_coeff"]):
        d.out_addr.coeff[i] = c
    d.combine, d.reduce, d.beta, d.n_epi = nest["combine"], nest["reduce"], nest["beta"], 0
    out.zero_()
    native.affine_nest(d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy(), native.last_nest_kernel()


@pytest.mark.parametrize("aligned", [False, True], ids=["ragged", "aligned"])
@pytest.mark.parametrize("seed", range(40))
def test_random_nest(seed, aligned, monkeypatch):
    native.init(0)
    rng = np.random.default_rng(1000 * int(aligned) + seed)
    nest = _random_nest(rng, aligned)
    bufs = [rng.integers(-3, 4, size=op["size"]).astype(np.float32) for op in nest["ops"]]
    dev = [torch.from_numpy(b).cuda() for b in bufs]
    out = torch.zeros(nest["out_size"], device="cuda")
    want = _numpy_eval(nest, bufs)
    fast, kind = _run(nest, dev, out)
    monkeypatch.setenv("LSB_NO_NEST_FAST", "1")
    gen, gkind = _run(nest, dev, out)
    assert gkind == 0 and kind != 0, (kind, gkind)
    assert np.array_equal(fast.view(np.uint32), gen.view(np.uint32)), f"fast (kernel {kind}) != general: {nest}"
    assert np.array_equal(np.nan_to_num(fast, nan=7e7), np.nan_to_num(want, nan=7e7)), f"kernel {kind}: {nest}"


def test_fuzz_reaches_every_fast_kernel():
    """The generator's shapes should exercise rows, vec4 and pool / transpose
    at least through the resized acceptance nests (test_gpu_nest_fast.py); here:
    rows and vec4 must both occur among the random nests."""
    native.init(0)
    kinds = set()
    for aligned, seed in itertools.product([False, True], range(40)):
        rng = np.random.default_rng(1000 * int(aligned) + seed)
        nest = _random_nest(rng, aligned)
        bufs = [torch.from_numpy(rng.integers(-3, 4, size=op["size"]).astype(np.float32)).cuda() for op in nest["ops"]]
        out = torch.zeros(nest["out_size"], device="cuda")
        kinds.add(_run(nest, bufs, out)[1])
    assert {1, 3} <= kinds, kinds
