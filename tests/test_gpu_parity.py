"""Parity of the CUDA path against the oracle and the reference's own outputs.

Every case goes through the drop-in surface (compile_graph -> execute, the
reference's compile-then-call contract, backend.py:121-161) and therefore
through the C ABI in liblsb.so.  Rules (BASELINE north_star):
  bitexact  max/min semirings: GPU f32 == float32(reference_eval) per element
            (and == the reference VM's bytes for C2);
  exact     small-integer inputs: every summation order is exact, so == too;
  tol       fp32 sum reductions: |d| <= 1e-5 + 1e-4|ref| per element for the
            configs; the reference's acceptance metric max|d|/max(|ref|,1)
            <= 1e-4 (test_acceptance.py:23) for the small semiring sweep;
  refmetric C5 (K = 16384): reference metric on sampled rows/cols.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import common
from paper_2205_00618_b200 import backend, native

pytestmark = pytest.mark.gpu

IDX = common.index()
SMALL = IDX["cases"]


def _run(graph_json: str, bufs: dict):
    k = backend.compile_graph(graph_json)
    got = {s: np.array(b, copy=True) for s, b in bufs.items()}
    backend.execute(k, got)
    return k, got


@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_small_case(case):
    gj = common.graph_json(case["graph"])
    ins, ref, vm = common.case_data(case)
    # alpha cases seed the output slot with C_in (stored among the inputs)
    k, got = _run(gj, ins)
    assert k.counters["launches"] >= 1
    sig = "sigmoid" in gj
    for slot, r in ref.items():
        ok, msg = common.check_case(case["rule"], got[slot], r, has_sigmoid=sig)
        assert ok, f"{case['name']} slot {slot}: {msg}"
        # where the reference VM itself is right (it miscompiles uneven vector
        # tails, SURVEY finding 3), the GPU must reproduce its bytes too
        if case["rule"] == "bitexact" and slot in vm and common.value_exact(vm[slot], r):
            assert np.array_equal(got[slot].reshape(vm[slot].shape), vm[slot]), "differs from VM"


TC_CASES = [c for c in SMALL if c["name"] in (
    "semiring_mul_add", "fma_node", "transposed_gemm", "kat_identity_operand", "kat_alpha1_beta0",
    "epi_beta_half_mul_add", "epi_beta_neg_mul_add", "epi_alpha_relu_pre_mul_add",
    "epi_alpha_sig_post_mul_add", "epi_post_relu_mul_add", "mlp_bias_relu_small",
    "mlp_alpha_relu_small", "mlp_bias_sigmoid_small", "acc_mm16", "acc_mm64",
    "conv_valid_small", "conv_pad1_small", "conv_stride2_small")]


@pytest.mark.parametrize("case", TC_CASES, ids=[c["name"] for c in TC_CASES])
def test_small_case_forced_tensor_core_path(case, monkeypatch):
    """The same fixtures through the 3xTF32 tcgen05 kernels (GEMM and
    im2col conv), which auto-selection only uses for large problems."""
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    gj = common.graph_json(case["graph"])
    ins, ref, _ = common.case_data(case)
    k, got = _run(gj, ins)
    for slot, r in ref.items():
        m = common.ref_metric(got[slot], r)
        assert m <= 1e-4, f"{case['name']}: metric {m}"
        if case["rule"] in ("tol", "exact"):
            assert common.strict_ok(got[slot], r).all(), case["name"]


CONV_CASES = [c for c in SMALL if c["name"] in ("conv_valid_small", "conv_pad1_small", "conv_stride2_small",
                                                 "acc_conv1d")]


@pytest.mark.parametrize("algo", ["tf32x3", "tf32x3_nhwc", "tf32x3_planar", "simt"])
@pytest.mark.parametrize("case", CONV_CASES, ids=[c["name"] for c in CONV_CASES])
def test_conv_cases_every_conv_kernel(case, algo, monkeypatch):
    """Each conv kernel (planar single-pass tensor-core kernel, NHWC-copy
    tensor-core kernel, SIMT) on the conv fixtures; kernels whose
    preconditions fail fall back (lsb_conv2d_nchw) and must still be right."""
    monkeypatch.setenv("LSB_GEMM_ALGO", algo)
    gj = common.graph_json(case["graph"])
    ins, ref, _ = common.case_data(case)
    k, got = _run(gj, ins)
    for slot, r in ref.items():
        assert common.ref_metric(got[slot], r) <= 1e-4, case["name"]
        if case["rule"] in ("tol", "exact"):
            assert common.strict_ok(got[slot], r).all(), case["name"]


@pytest.mark.parametrize("algo", ["tf32x3", "tf32x3_nhwc", "tf32x3_planar", "simt"])
def test_c3_every_conv_kernel(algo, monkeypatch):
    """C3 (guarded-view form) through each conv kernel, all 8 images checked
    against f64 (numpy restatement of the conv, SURVEY §8(c) rule)."""
    monkeypatch.setenv("LSB_GEMM_ALGO", algo)
    cfg = common.config("C3")
    bufs = common.config_inputs("C3g")
    k, got = _run(common.graph_json(cfg["graph_guarded"]), bufs)
    o = got[2].reshape(8, 64, 56, 56)
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    ref0 = d["ref_img0"].astype(np.float64).reshape(64, 56, 56)
    assert common.strict_ok(o[0], ref0).all()
    ref = _conv_f64(bufs[0], bufs[1], 1)
    ok = common.strict_ok(o, ref)
    assert ok.all(), (algo, float(ok.mean()), common.ref_metric(o, ref))


def _conv_f64(x, w, pad):
    """f64 NCHW stride-1 conv: the (mul, add) contraction reference_eval
    evaluates, summed tap by tap (exact enough: f64 error << tolerance)."""
    n, c, h, wd = x.shape
    co, _, r, s = w.shape
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    ho, wo = h + 2 * pad - r + 1, wd + 2 * pad - s + 1
    out = np.zeros((n, co, ho, wo))
    w64 = w.astype(np.float64)
    for i in range(r):
        for j in range(s):
            out += np.einsum("nchw,oc->nohw", xp[:, :, i:i + ho, j:j + wo], w64[:, :, i, j], optimize=True)
    return out


def test_inputs_not_mutated_and_output_inserted():
    case = next(c for c in SMALL if c["name"] == "semiring_mul_add")
    ins, ref, _ = common.case_data(case)
    before = {s: a.copy() for s, a in ins.items()}
    k = backend.compile_graph(common.graph_json(case["graph"]))
    bufs = dict(ins)
    backend.execute(k, bufs)
    for s in before:
        assert np.array_equal(before[s], ins[s])
    assert 2 in bufs and bufs[2].shape == (37, 53)


def test_shape_mismatch_raises():
    case = next(c for c in SMALL if c["name"] == "semiring_mul_add")
    ins, _, _ = common.case_data(case)
    k = backend.compile_graph(common.graph_json(case["graph"]))
    with pytest.raises(backend.ShapeMismatch):
        backend.execute(k, {0: ins[0]})
    with pytest.raises(backend.ShapeMismatch):
        backend.execute(k, {0: ins[0], 1: ins[1][:3]})


# ---------------------------------------------------------------- BASELINE configs

def test_c1_gemm_256():
    cfg = common.config("C1")
    bufs = common.config_inputs("C1")
    assert common.sha(bufs[0]) == cfg["in_sha"]["0"]
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    _, got = _run(common.graph_json(cfg["graph"]), bufs)
    c = got[2].reshape(256, 256)
    assert common.strict_ok(c, d["ref_2"]).all(), common.ref_metric(c, d["ref_2"])


def test_c2_maxplus_bit_exact_vs_reference_vm():
    cfg = common.config("C2")
    bufs = common.config_inputs("C2")
    assert common.sha(bufs[0]) == cfg["in_sha"]["0"]
    _, got = _run(common.graph_json(cfg["graph"]), bufs)
    c = got[2].reshape(1024, 1024)
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    assert np.array_equal(c[:64], d["ref_rows0_64"].astype(np.float32))
    # the reference VM's full 1024x1024 output, byte for byte
    assert common.sha(c) == cfg["vm_out_sha"]


@pytest.mark.parametrize("name", ["C3", "C3g"])
def test_c3_conv(name):
    """All 8 images: image 0 against the stored reference_eval output, every
    image against the oracle restatement (f64) restricted to that image."""
    cfg = common.config("C3")
    bufs = common.config_inputs(name)
    graph = common.graph_json(cfg["graph"] if name == "C3" else cfg["graph_guarded"])
    k, got = _run(graph, bufs)
    assert k.plan.steps[0].kind == "conv"
    o = got[2].reshape(8, 64, 56, 56)
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    ref0 = d["ref_img0"].astype(np.float64).reshape(64, 56, 56)
    assert common.strict_ok(o[0], ref0).all()
    from oracle import oracle as O
    from paper_2205_00618_b200.graph import Graph
    g = Graph.from_json(graph)
    nvar = [v.id for v in g.vars.values() if v.name == "n"][0]
    for img in range(8):
        ref = O.reference_eval(g, bufs, restrict={nvar: np.array([img])})[2]
        ok = common.strict_ok(o[img:img + 1], ref)
        assert ok.all(), (img, float(ok.mean()), common.ref_metric(o[img:img + 1], ref))


def _f64_gemm_rows(X, W, b=None, relu=False, block=512):
    out = np.empty((X.shape[0], W.shape[1]), np.float64)
    W64 = W.astype(np.float64)
    for r in range(0, X.shape[0], block):
        y = X[r:r + block].astype(np.float64) @ W64
        if b is not None:
            y += b.astype(np.float64)
        out[r:r + block] = np.maximum(y, 0.0) if relu else y
    return out


@pytest.mark.parametrize("bias_nonzero", [False, True])
def test_c4_mlp_bias_relu(bias_nonzero):
    """All 4096 x 4096 outputs against an f64 restatement (rows 0-63 also
    against the stored reference_eval output)."""
    cfg = common.config("C4")
    bufs = common.config_inputs("C4", bias_nonzero)
    k, got = _run(common.graph_json(cfg["graph"]), bufs)
    assert len(k.plan.steps) == 1 and k.plan.steps[0].kind == "gemm"   # bias+ReLU fused
    y = got[3].reshape(4096, 4096)
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    ref = d["ref_rows0_64_bnz" if bias_nonzero else "ref_rows0_64_b0"]
    assert common.strict_ok(y[:64], ref).all()
    want = _f64_gemm_rows(bufs[0], bufs[1], bufs[2], relu=True)
    ok = common.strict_ok(y, want)
    assert ok.all(), (float(ok.mean()), common.ref_metric(y, want))


def test_c4_alpha_form():
    cfg = common.config("C4")
    bufs = common.config_inputs("C4a", bias_nonzero=True)
    k, got = _run(common.graph_json(cfg["graph_alpha"]), bufs)
    y = got[2].reshape(4096, 4096)
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    assert common.strict_ok(y[:64], d["ref_rows0_64_bnz"]).all()


@pytest.mark.slow
def test_c5_gemm_16384_full():
    """Every one of the 16384^2 outputs against an f64 GEMM (computed on the
    device in torch float64 -- the f64 restatement of reference_eval's
    (mul, add) contraction).  Gate: the reference metric, per
    element as the reference computes it, max(|d|/max(|ref|,1)) <= 1e-4
    (measured 8.5e-5 over all 268M outputs; the VM's own is 3.2e-4 on rows
    0-7); the strict per-element pass fraction is
    recorded next to the reference VM's own on rows 0-7 (the VM fails the
    strict rule on ~0.6 % at K = 16384) and must not be worse than it."""
    import json
    import torch
    cfg = common.config("C5")
    bufs = common.config_inputs("C5")
    _, got = _run(common.graph_json(cfg["graph"]), bufs)
    C = got[2].reshape(16384, 16384)
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    ref8 = d["ref_rows0_8"]
    vm = float(common.strict_ok(d["vm_rows0_8"], ref8).mean())
    dev = torch.device("cuda", 0)
    A = torch.from_numpy(bufs[0]).to(dev).double()
    B = torch.from_numpy(bufs[1]).to(dev).double()
    Cg = torch.from_numpy(C).to(dev)
    worst, npass, amax, tot, elem = 0.0, 0, 0.0, 0, 0.0
    for r in range(0, 16384, 2048):
        ref = A[r:r + 2048] @ B
        dd = (Cg[r:r + 2048].double() - ref).abs()
        worst = max(worst, float(dd.max()))
        amax = max(amax, float(ref.abs().max()))
        # the reference's acceptance formula, per element (test_acceptance.py:57-58)
        elem = max(elem, float((dd / ref.abs().clamp(min=1.0)).max()))
        npass += int((dd <= 1e-5 + 1e-4 * ref.abs()).sum())
        tot += ref.numel()
    metric = worst / max(amax, 1.0)
    strict = npass / tot
    rec = {"config": "C5", "elements": tot, "ref_metric": elem, "max_err_rel_max_ref": metric,
           "strict_pass": strict,
           "vm_strict_pass_rows0_8": vm, "ours_strict_pass_rows0_8": float(common.strict_ok(C[:8], ref8).mean()),
           "ours_ref_metric_rows0_8": common.ref_metric(C[:8], ref8),
           "vm_ref_metric_rows0_8": common.ref_metric(d["vm_rows0_8"], ref8)}
    print("C5 parity:", json.dumps(rec))
    out = os.environ.get("LSB_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)
    assert elem <= 1e-4, rec
    assert strict >= vm, rec


def test_launch_accounting():
    n0 = native.launch_count()
    case = next(c for c in SMALL if c["name"] == "acc_mlp3")
    ins, _, _ = common.case_data(case)
    k, _ = _run(common.graph_json(case["graph"]), ins)
    assert native.launch_count() - n0 == len(k.plan.steps) == 3
