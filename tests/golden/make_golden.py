"""Generate the parity fixtures under tests/golden/ from the REAL reference.

Run here (dev container, where /root/reference exists):

    python tests/golden/make_golden.py

It imports loopsmith from /root/reference/pkg/src (read-only) and writes:

  graphs/<name>.json   canonical graph JSON from loopsmith.serialize.dumps
                       (the exact bytes the reference would save)
  data/<name>.npz      inputs, reference_eval outputs (f64, "ref_<slot>") and
                       reference-VM outputs (f32, "vm_<slot>") for small cases
  index.json           case list: graph file, parity rule, seeds, input and
                       output digests for the BASELINE-sized configs

Nothing on the GPU box reads /root/reference: the tests only read these files.
Seeded inputs follow SURVEY.md §8(d) (np.random.default_rng(seed), operands
drawn in listed order); the small cases use the reference tests' small-integer
convention (op_graphs.random_inputs, lo=-3, hi=4) or uniform floats.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path[:0] = [REF_SRC, REF_TESTS]

import loopsmith as ls  # noqa: E402
from loopsmith import schedule as sch  # noqa: E402
from loopsmith import serialize  # noqa: E402
from loopsmith.ir import Arith, DFG, Read, VirtualBuffer, Write  # noqa: E402
import op_graphs  # noqa: E402
from schedule_fuzz import random_actions  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GDIR = os.path.join(HERE, "graphs")
DDIR = os.path.join(HERE, "data")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


# ---------------------------------------------------------------- graph builders

def reorder_all(g, order_names):
    """test_backend.py:16-27 idiom: apply one global order, filtered per node."""
    for node in g:
        names = [v.name for v in node.order]
        sch.apply_action(g, sch.ReorderAction(
            node.id, [nm for nm in order_names if nm in names]
            + [nm for nm in names if nm not in order_names]))


def gemm(m, k, n, sched=True, alpha=0.0, beta=1.0):
    g = ls.matmul_graph(m, k, n, alpha=alpha, beta=beta)
    if sched:
        sch.split(g, sch.find_var(g, "m"), min(4, m))
        sch.split(g, sch.find_var(g, "n"), min(64, n))
        reorder_all(g, ["m_o", "n_o", "k", "m_i", "n_i"])
    return g


def semiring(m, k, n, combine="add", reduce="max", sched=True, beta=1.0,
             alpha=0.0, pre="identity", post="identity"):
    b = ls.GraphBuilder()
    vm_, vk, vn = b.var("m", m), b.var("k", k), b.var("n", n)
    a, bb = b.input("a", [vm_, vk]), b.input("b", [vk, vn])
    rhs = a[vm_, vk] + bb[vk, vn] if combine == "add" else a[vm_, vk] * bb[vk, vn]
    c = b.contract("c", (vm_, vn), rhs, op_pair=(reduce, combine), beta=beta,
                   alpha=alpha, pre=pre, post=post)
    b.output(c)
    g = b.build()
    if sched:
        sch.split(g, sch.find_var(g, "m"), min(4, m))
        sch.split(g, sch.find_var(g, "n"), min(64, n))
        reorder_all(g, ["m_o", "n_o", "k", "m_i", "n_i"])
    return g


def raw_combine(m, k, n, combine="max", reduce="add"):
    """Combine ops the frontend cannot spell (max/min): built on the IR."""
    g = DFG()
    vm_, vk, vn = ls.Var("m", m), ls.Var("k", k), ls.Var("n", n)
    a = g.add(Read(0), (), VirtualBuffer("a", (vm_, vk)))
    b = g.add(Read(1), (), VirtualBuffer("b", (vk, vn)))
    t = g.add(Arith(combine), (a.id, b.id), VirtualBuffer("t", (vm_, vk, vn)))
    c = g.add(Arith(reduce), (t.id,), VirtualBuffer("c", (vm_, vn)))
    g.add(Write(2), (c.id,), VirtualBuffer("c_out", (vm_, vn)))
    assert not ls.validate(g)
    return g


def fma_node(m, k, n):
    """A single 2-input 'fma' node (ir.py:190) that reduces directly."""
    g = DFG()
    vm_, vk, vn = ls.Var("m", m), ls.Var("k", k), ls.Var("n", n)
    a = g.add(Read(0), (), VirtualBuffer("a", (vm_, vk)))
    b = g.add(Read(1), (), VirtualBuffer("b", (vk, vn)))
    c = g.add(Arith("fma"), (a.id, b.id), VirtualBuffer("c", (vm_, vn)))
    g.add(Write(2), (c.id,), VirtualBuffer("c_out", (vm_, vn)))
    assert not ls.validate(g)
    return g


def conv(n, ci, h, w, co, r=3, s=3, stride=1, sched=True, guarded_pad=0):
    """NCHW direct conv.  guarded_pad=0: valid conv over an input of spatial
    size (h-1)*stride+r (host-padded form).  guarded_pad=p: conv over an
    unpadded input through a guarded view with offset -p (oob 0)."""
    b = ls.GraphBuilder()
    vn, vci, vco = b.var("n", n), b.var("ci", ci), b.var("co", co)
    vh, vw, vkh, vkw = b.var("h", h), b.var("w", w), b.var("kh", r), b.var("kw", s)
    if guarded_pad:
        hin, win = h * stride - 2 * guarded_pad + r - 1, w * stride - 2 * guarded_pad + s - 1
    else:
        hin, win = (h - 1) * stride + r, (w - 1) * stride + s
    x = b.input("x", [vn, vci, b.var("hp", hin), b.var("wp", win)])
    wt = b.input("wt", [vco, vci, vkh, vkw])
    if guarded_pad:
        idx = (vn, vci, vh * stride + vkh - guarded_pad, vw * stride + vkw - guarded_pad)
        view = b._emit_view(x, idx, guarded=True, oob=0.0)
        from loopsmith.frontend import Tensor
        xv = Tensor(b, "xv", b.dfg[view].output.dims, b.dfg[view])
        rhs = xv[tuple(b.dfg[view].output.dims)] * wt[vco, vci, vkh, vkw]
    else:
        rhs = x[vn, vci, vh * stride + vkh, vw * stride + vkw] * wt[vco, vci, vkh, vkw]
    o = b.contract("o", (vn, vco, vh, vw), rhs)
    b.output(o)
    g = b.build()
    if sched:
        sch.split(g, sch.find_var(g, "co"), min(8, co))
        sch.split(g, sch.find_var(g, "w"), min(8, w))
        reorder_all(g, ["n", "h", "co_o", "w_o", "ci", "kh", "kw", "co_i", "w_i"])
    return g


def mlp_bias_relu(bsz, k, n, sched=True, alpha_form=False, post="relu"):
    """C4: Y = ReLU(X.W + b).  Two-statement form (h then h+bias with post),
    or the alpha form (bias pre-seeded into the output slot, alpha=1)."""
    g = ls.GraphBuilder()
    vb, vk, vn = g.var("b", bsz), g.var("k", k), g.var("n", n)
    x, w = g.input("x", [vb, vk]), g.input("w", [vk, vn])
    if alpha_form:
        y = g.contract("y", (vb, vn), x[vb, vk] * w[vk, vn], post=post, alpha=1.0)
    else:
        bias = g.input("bias", [vn])
        h = g.contract("h", (vb, vn), x[vb, vk] * w[vk, vn])
        y = g.contract("y", (vb, vn), h[vb, vn] + bias[vn], post=post)
    g.output(y)
    dfg = g.build()
    if sched:
        sch.split(dfg, sch.find_var(dfg, "b"), min(4, bsz))
        sch.split(dfg, sch.find_var(dfg, "n"), min(64, n))
        reorder_all(dfg, ["b_o", "n_o", "k", "b_i", "n_i"])
    return dfg


def batched_gemm(bt, m, k, n):
    b = ls.GraphBuilder()
    vb, vm_, vk, vn = b.var("bt", bt), b.var("m", m), b.var("k", k), b.var("n", n)
    a, bb = b.input("a", [vb, vm_, vk]), b.input("b", [vb, vk, vn])
    c = b.contract("c", (vb, vm_, vn), a[vb, vm_, vk] * bb[vb, vk, vn])
    b.output(c)
    return b.build()


def transposed_gemm(m, k, n):
    """C[m,n] = sum_k A[k,m] * B[n,k]: both operands transposed."""
    b = ls.GraphBuilder()
    vm_, vk, vn = b.var("m", m), b.var("k", k), b.var("n", n)
    a, bb = b.input("a", [vk, vm_]), b.input("b", [vn, vk])
    c = b.contract("c", (vm_, vn), a[vk, vm_] * bb[vn, vk])
    b.output(c, dims=[vn, vm_])   # stored transposed too
    return b.build()


# ---------------------------------------------------------------- inputs

def uniform_inputs(dfg, seed, lo, hi, order=None):
    rng = np.random.default_rng(seed)
    shapes = ls.slot_shapes(dfg)
    ins = sorted(n.kind.slot for n in dfg if isinstance(n.kind, Read))
    return {s: rng.uniform(lo, hi, shapes[s]).astype(np.float32) for s in (order or ins)}


def int_inputs(dfg, seed):
    return op_graphs.random_inputs(dfg, np.random.default_rng(seed))


def run_vm(dfg, bufs, target=ls.avx512_like):
    kern = ls.compile_tree(ls.lower(dfg), target())
    got = {s: b.copy() for s, b in bufs.items()}
    ls.execute(kern, got)
    outs = {n.kind.slot for n in dfg if isinstance(n.kind, Write)}
    return {s: got[s].reshape(ls.slot_shapes(dfg)[s]).astype(np.float32) for s in outs}


# ---------------------------------------------------------------- main

INDEX: list[dict] = []


def save_graph(name, dfg):
    path = os.path.join(GDIR, f"{name}.json")
    with open(path, "w") as f:
        f.write(serialize.dumps(dfg))
    return f"graphs/{name}.json"


def small_case(name, dfg, bufs, rule, vm=True, target=ls.avx512_like, note="", seed_out=None):
    gfile = save_graph(name, dfg)
    ref = ls.reference_eval(dfg, bufs)
    arrays = {f"in_{s}": np.asarray(b) for s, b in bufs.items()}
    for s, r in ref.items():
        arrays[f"ref_{s}"] = r
    if vm:
        for s, v in run_vm(dfg, bufs, target).items():
            arrays[f"vm_{s}"] = v
    np.savez_compressed(os.path.join(DDIR, f"{name}.npz"), **arrays)
    INDEX.append({"name": name, "graph": gfile, "data": f"data/{name}.npz",
                  "rule": rule, "size": "small", "note": note})


def main():
    os.makedirs(GDIR, exist_ok=True)
    os.makedirs(DDIR, exist_ok=True)
    t0 = time.time()

    # --- the reference's own acceptance operator set (op_graphs.py:89-98),
    #     integer inputs (exact under any summation order)
    for i, (name, build) in enumerate(op_graphs.ACCEPTANCE_OPS.items()):
        dfg = build()
        rule = "exact"
        small_case(f"acc_{name}", dfg, int_inputs(dfg, 100 + i), rule,
                   note="op_graphs.ACCEPTANCE_OPS, default schedule")
    # same ops under random legal schedules (schedule invariance)
    rng = random.Random(2024)
    for name, build in op_graphs.ACCEPTANCE_OPS.items():
        for j in range(20):
            dfg = build()
            random_actions(dfg, rng, max_splits=3)
            small_case(f"fuzz_{name}_{j}", dfg, int_inputs(dfg, 500 + j), "exact", vm=False,
                       note="schedule_fuzz.random_actions(seed 2024)")

    # --- KATs pinned by the reference tests
    dfg = semiring(4, 4, 4, "add", "max", sched=False)
    rng_ = np.random.default_rng(2)
    a = rng_.integers(-5, 6, (4, 4)).astype(np.float32)
    b = rng_.integers(-5, 6, (4, 4)).astype(np.float32)
    small_case("kat_tropical_4", dfg, {0: a, 1: b}, "bitexact",
               note="test_feedback.py:93-110 brute-force tropical KAT")
    dfg = op_graphs.maxpool2x2(4)
    small_case("kat_maxpool_ramp", dfg, {0: np.arange(16, dtype=np.float32).reshape(4, 4)},
               "bitexact", target=ls.avx2_like, note="test_feedback.py:113-122 -> [[5,7],[13,15]]")
    dfg = ls.matmul_graph(4, 4, 4)
    rng_ = np.random.default_rng(0)
    small_case("kat_identity_operand", dfg,
               {0: rng_.integers(-3, 4, (4, 4)).astype(np.float32), 1: np.eye(4, dtype=np.float32)},
               "exact", note="test_feedback.py:73-79")
    dfg = ls.matmul_graph(4, 4, 4, alpha=1.0, beta=0.0)
    rng_ = np.random.default_rng(1)
    small_case("kat_alpha1_beta0", dfg,
               {0: rng_.random((4, 4)).astype(np.float32), 1: rng_.random((4, 4)).astype(np.float32),
                2: rng_.random((4, 4)).astype(np.float32)},
               "tol", note="test_feedback.py:82-90: output == prior contents")

    # --- semiring operator pairs on ragged shapes (frontend-expressible)
    for comb in ("mul", "add"):
        for red in ("add", "max", "min", "mul"):
            dfg = semiring(37, 29, 53, comb, red)
            lo, hi = (0.9, 1.1) if red == "mul" else (-10.0, 10.0)
            bufs = uniform_inputs(dfg, 11, lo, hi)
            rule = "bitexact" if red in ("max", "min") and comb == "add" else "tol"
            small_case(f"semiring_{comb}_{red}", dfg, bufs, rule,
                       note="ragged 37x29x53, split m4 n64 schedule")
    for comb, red in (("max", "add"), ("min", "add"), ("max", "min"), ("min", "max")):
        dfg = raw_combine(33, 17, 45, comb, red)
        small_case(f"rawcomb_{comb}_{red}", dfg, uniform_inputs(dfg, 12, -4.0, 4.0),
                   "bitexact" if red in ("max", "min") else "tol", note="IR-built combine op")
    dfg = fma_node(31, 19, 41)
    small_case("fma_node", dfg, uniform_inputs(dfg, 13, -1.0, 1.0), "tol", note="single fma node")
    # alpha / beta / pre / post variants
    for tag, kw in (("beta_half", dict(beta=0.5)), ("beta_neg", dict(beta=-2.0)),
                    ("beta_zero", dict(beta=0.0)),
                    ("alpha_relu_pre", dict(alpha=1.5, pre="relu")),
                    ("alpha_sig_post", dict(alpha=-0.5, post="sigmoid")),
                    ("post_relu", dict(post="relu"))):
        for comb, red in (("mul", "add"), ("add", "max")):
            dfg = semiring(24, 40, 70, comb, red, **kw)
            bufs = uniform_inputs(dfg, 14, -2.0, 2.0)
            if kw.get("alpha"):
                bufs[2] = np.random.default_rng(15).uniform(-3, 3, (24, 70)).astype(np.float32)
            rule = "bitexact" if red == "max" and not kw.get("post") == "sigmoid" else "tol"
            small_case(f"epi_{tag}_{comb}_{red}", dfg, bufs, rule, note=str(kw))
    # layouts
    dfg = batched_gemm(3, 20, 36, 28)
    small_case("batched_gemm", dfg, uniform_inputs(dfg, 16, -1, 1), "tol")
    dfg = transposed_gemm(45, 33, 21)
    small_case("transposed_gemm", dfg, uniform_inputs(dfg, 17, -1, 1), "tol")
    # conv variants (small), C4-like variants (small)
    dfg = conv(2, 3, 10, 10, 4)
    small_case("conv_valid_small", dfg, uniform_inputs(dfg, 18, -1, 1), "tol")
    dfg = conv(2, 5, 9, 11, 6, guarded_pad=1)
    small_case("conv_pad1_small", dfg, uniform_inputs(dfg, 19, -1, 1), "tol", target=ls.avx2_like)
    dfg = conv(1, 4, 6, 7, 5, stride=2, sched=False)
    small_case("conv_stride2_small", dfg, uniform_inputs(dfg, 20, -1, 1), "tol")
    dfg = mlp_bias_relu(48, 40, 96)
    rng_ = np.random.default_rng(21)
    bufs = {0: rng_.normal(0, 1, (48, 40)).astype(np.float32),
            1: rng_.normal(0, 1, (40, 96)).astype(np.float32),
            2: rng_.normal(0, 1, (96,)).astype(np.float32)}
    small_case("mlp_bias_relu_small", dfg, bufs, "tol", note="nonzero bias")
    dfg = mlp_bias_relu(40, 24, 72, alpha_form=True)
    rng_ = np.random.default_rng(22)
    bias = rng_.normal(0, 1, (72,)).astype(np.float32)
    bufs = {0: rng_.normal(0, 1, (40, 24)).astype(np.float32),
            1: rng_.normal(0, 1, (24, 72)).astype(np.float32),
            2: np.broadcast_to(bias, (40, 72)).astype(np.float32).copy()}
    small_case("mlp_alpha_relu_small", dfg, bufs, "tol", note="alpha form, bias pre-seeded")
    dfg = mlp_bias_relu(36, 20, 50, post="sigmoid")
    rng_ = np.random.default_rng(23)
    bufs = {0: rng_.normal(0, 1, (36, 20)).astype(np.float32),
            1: rng_.normal(0, 1, (20, 50)).astype(np.float32),
            2: rng_.normal(0, 1, (50,)).astype(np.float32)}
    small_case("mlp_bias_sigmoid_small", dfg, bufs, "tol")

    # --- BASELINE configs: graphs + digests + slices
    configs = []
    # C1 full (reference_eval runs directly)
    dfg = gemm(256, 256, 256)
    bufs = uniform_inputs(dfg, 0, -1.0, 1.0)
    gfile = save_graph("C1", dfg)
    ref = ls.reference_eval(dfg, bufs)
    vmo = run_vm(dfg, bufs)
    np.savez_compressed(os.path.join(DDIR, "C1.npz"), ref_2=ref[2].astype(np.float64),
                        vm_2=vmo[2])
    configs.append({"name": "C1", "graph": gfile, "data": "data/C1.npz", "seed": 0,
                    "dist": ["uniform", -1.0, 1.0], "rule": "tol",
                    "in_sha": {str(s): sha(b) for s, b in bufs.items()}})
    # C2 max-plus: VM full output digest (bit-exact target) + reference slice
    dfg = semiring(1024, 1024, 1024, "add", "max")
    bufs = uniform_inputs(dfg, 1, -10.0, 10.0)
    gfile = save_graph("C2", dfg)
    t = time.time()
    vmo = run_vm(dfg, bufs)
    vm_s = time.time() - t
    sl = semiring(64, 1024, 1024, "add", "max", sched=False)
    ref_sl = ls.reference_eval(sl, {0: bufs[0][:64], 1: bufs[1]})[2]
    assert np.array_equal(vmo[2][:64], ref_sl.astype(np.float32)), "VM != f32(ref) on C2 slice"
    np.savez_compressed(os.path.join(DDIR, "C2.npz"), ref_rows0_64=ref_sl, vm_rows0_64=vmo[2][:64])
    configs.append({"name": "C2", "graph": gfile, "data": "data/C2.npz", "seed": 1,
                    "dist": ["uniform", -10.0, 10.0], "rule": "bitexact",
                    "in_sha": {str(s): sha(b) for s, b in bufs.items()},
                    "vm_out_sha": sha(vmo[2]), "vm_seconds_here": vm_s})
    # C3 conv (host-padded form and guarded-view form)
    for name, gp in (("C3", 0), ("C3g", 1)):
        dfg = conv(8, 64, 56, 56, 64, guarded_pad=gp)
        save_graph(name, dfg)
    rng_ = np.random.default_rng(2)
    x = rng_.uniform(-1.0, 1.0, (8, 64, 56, 56)).astype(np.float32)
    w = rng_.normal(0.0, np.sqrt(2.0 / 576.0), (64, 64, 3, 3)).astype(np.float32)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    one = conv(1, 64, 56, 56, 64, guarded_pad=0, sched=False)
    ref0 = ls.reference_eval(one, {0: xp[:1], 1: w})
    one_sched = conv(1, 64, 56, 56, 64, guarded_pad=0)
    vm0 = run_vm(one_sched, {0: xp[:1], 1: w}, ls.avx2_like)
    np.savez_compressed(os.path.join(DDIR, "C3.npz"), ref_img0=ref0[2].astype(np.float32),
                        vm_img0=vm0[2])
    configs.append({"name": "C3", "graph": "graphs/C3.json", "graph_guarded": "graphs/C3g.json",
                    "data": "data/C3.npz", "seed": 2, "rule": "tol",
                    "in_sha": {"x": sha(x), "w": sha(w)}})
    # C4 MLP bias+ReLU (b = 0, plus nonzero-bias parity run)
    dfg = mlp_bias_relu(4096, 1024, 4096)
    save_graph("C4", dfg)
    save_graph("C4a", mlp_bias_relu(4096, 1024, 4096, alpha_form=True))
    rng_ = np.random.default_rng(3)
    X = rng_.normal(0, 0.02, (4096, 1024)).astype(np.float32)
    W = rng_.normal(0, 0.02, (1024, 4096)).astype(np.float32)
    bnz = rng_.normal(0, 0.02, (4096,)).astype(np.float32)
    rows = np.arange(64)
    sl = mlp_bias_relu(64, 1024, 4096, sched=False)
    ref0 = ls.reference_eval(sl, {0: X[:64], 1: W, 2: np.zeros(4096, np.float32)})[3]
    refb = ls.reference_eval(sl, {0: X[:64], 1: W, 2: bnz})[3]
    vmsl = run_vm(mlp_bias_relu(64, 1024, 4096), {0: X[:64], 1: W, 2: bnz})[3]
    np.savez_compressed(os.path.join(DDIR, "C4.npz"), ref_rows0_64_b0=ref0, ref_rows0_64_bnz=refb,
                        vm_rows0_64_bnz=vmsl)
    configs.append({"name": "C4", "graph": "graphs/C4.json", "graph_alpha": "graphs/C4a.json",
                    "data": "data/C4.npz", "seed": 3, "rule": "tol",
                    "in_sha": {"x": sha(X), "w": sha(W), "bias_nz": sha(bnz)}})
    # C5 large GEMM: graph + input digests + an 8-row VM slice (strict-rule comparison)
    dfg = gemm(16384, 16384, 16384)
    save_graph("C5", dfg)
    rng_ = np.random.default_rng(4)
    A = rng_.uniform(-1, 1, (16384, 16384)).astype(np.float32)
    B = rng_.uniform(-1, 1, (16384, 16384)).astype(np.float32)
    sl = gemm(8, 16384, 16384)
    vm8 = run_vm(sl, {0: A[:8], 1: B})[2]
    ref8 = A[:8].astype(np.float64) @ B.astype(np.float64)
    np.savez_compressed(os.path.join(DDIR, "C5.npz"), vm_rows0_8=vm8, ref_rows0_8=ref8)
    configs.append({"name": "C5", "graph": "graphs/C5.json", "data": "data/C5.npz", "seed": 4,
                    "dist": ["uniform", -1.0, 1.0], "rule": "refmetric",
                    "in_sha": {"0": sha(A), "1": sha(B)}})

    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump({"generated_by": "tests/golden/make_golden.py",
                   "reference": "loopsmith 0.1.0 @ /root/reference/pkg/src",
                   "numpy": np.__version__, "cases": INDEX, "configs": configs}, f, indent=1)
    print(f"wrote {len(INDEX)} small cases + {len(configs)} configs in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
