"""Pin the oracle before trusting it (CPU only).

* oracle.reference_eval (f64 restatement of feedback.py:69-170) must equal the
  real reference_eval outputs stored by tests/golden/make_golden.py, exactly.
* oracle/vmport.c (C restatement of the VM's f32 arithmetic) must equal the
  real reference VM outputs bit for bit on the BASELINE configs.
* the seeded config inputs must reproduce the digests recorded at generation.
"""

from __future__ import annotations

import numpy as np
import pytest

import common
from oracle import oracle as O
from oracle import vmport
from paper_2205_00618_b200.graph import Graph

IDX = common.index()


@pytest.mark.parametrize("case", IDX["cases"], ids=[c["name"] for c in IDX["cases"]])
def test_restatement_equals_reference_eval(case):
    g = Graph.from_json(common.graph_json(case["graph"]))
    ins, ref, _ = common.case_data(case)
    out = O.reference_eval(g, ins)
    for slot, r in ref.items():
        assert np.array_equal(out[slot].reshape(r.shape), r), case["name"]


def test_restriction_and_chunking_match_full_eval():
    case = next(c for c in IDX["cases"] if c["name"] == "semiring_add_max")
    g = Graph.from_json(common.graph_json(case["graph"]))
    ins, ref, _ = common.case_data(case)
    m = [v.id for v in g.vars.values() if v.name == "m"][0]
    rows = np.array([0, 5, 36])
    old = O.CHUNK_ELEMS
    O.CHUNK_ELEMS = 64          # force many reduction chunks
    try:
        out = O.reference_eval(g, ins, restrict={m: rows})
    finally:
        O.CHUNK_ELEMS = old
    assert np.array_equal(out[2], ref[2][rows])


def test_c2_slice_restatement_matches_reference():
    cfg = common.config("C2")
    bufs = common.config_inputs("C2")
    g = Graph.from_json(common.graph_json(cfg["graph"]))
    m = [v.id for v in g.vars.values() if v.name == "m"][0]
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    out = O.reference_eval(g, bufs, restrict={m: np.arange(8)})
    assert np.array_equal(out[2], d["ref_rows0_64"][:8])


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5"])
def test_config_input_digests(name):
    if name == "C5":
        pytest.skip("2 GiB of inputs; digest checked in the GPU parity test")
    cfg = common.config(name)
    bufs = common.config_inputs(name, bias_nonzero=True)
    if name == "C4":
        assert common.sha(bufs[0]) == cfg["in_sha"]["x"]
        assert common.sha(bufs[2]) == cfg["in_sha"]["bias_nz"]
    else:
        for s, h in cfg["in_sha"].items():
            assert common.sha(bufs[int(s)]) == h


def test_vmport_bit_exact_vs_reference_vm_c1():
    cfg = common.config("C1")
    bufs = common.config_inputs("C1")
    d = np.load(common.GOLDEN + "/" + cfg["data"])
    assert np.array_equal(vmport.gemm(bufs[0], bufs[1]), d["vm_2"].reshape(256, 256))


def test_vmport_bit_exact_vs_reference_vm_c2_full():
    cfg = common.config("C2")
    bufs = common.config_inputs("C2")
    assert common.sha(vmport.gemm(bufs[0], bufs[1], "add", "max")) == cfg["vm_out_sha"]


def test_vmport_bit_exact_vs_reference_vm_c3_image0():
    d = np.load(common.GOLDEN + "/" + common.config("C3")["data"])
    bufs = common.config_inputs("C3g")
    o = vmport.conv2d(bufs[0], bufs[1], pad=1, images=(0, 1))
    assert np.array_equal(o[0], d["vm_img0"].reshape(64, 56, 56))


def test_vmport_bit_exact_vs_reference_vm_c4_rows():
    d = np.load(common.GOLDEN + "/" + common.config("C4")["data"])
    bufs = common.config_inputs("C4", bias_nonzero=True)
    y = vmport.gemm(bufs[0], bufs[1], bias=bufs[2], post="relu", rows=(0, 64))
    assert np.array_equal(y[:64], d["vm_rows0_64_bnz"].reshape(64, 4096))


def test_vmport_small_semirings_match_vm():
    for name in ("semiring_add_max", "semiring_add_min", "semiring_mul_add"):
        case = next(c for c in IDX["cases"] if c["name"] == name)
        ins, _, vm = common.case_data(case)
        comb, red = name.split("_")[1:]
        got = vmport.gemm(ins[0], ins[1], comb, red)
        assert np.array_equal(got, vm[2].reshape(got.shape)), name


def test_parity_rules():
    ref = np.array([[0.0, 2.0], [np.inf, -3.0]])
    assert common.check_case("bitexact", ref.astype(np.float32), ref)[0]
    bad = ref.copy()
    bad[0, 1] = 2.0 + 1e-3
    assert not common.check_case("tol", bad, ref)[0]
    assert O.ref_metric(ref, ref) == 0.0
    assert O.strict_ok(ref, ref).all()
