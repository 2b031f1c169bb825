"""Planner / drop-in surface on CPU: every reference graph plans onto the
kernel set, analytics equal the reference's, errors use the reference's
exception classes.  No kernel runs."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

import common
from paper_2205_00618_b200 import backend
from paper_2205_00618_b200.graph import Graph, GraphError
from paper_2205_00618_b200.planner import plan_graph

IDX = common.index()
ALL = IDX["cases"] + IDX["configs"]
REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF_SRC)


@pytest.mark.parametrize("case", ALL, ids=[c["name"] for c in ALL])
def test_every_golden_graph_plans(case):
    plan = plan_graph(common.graph_json(case["graph"]))
    assert plan.steps
    covered = {n for s in plan.steps for n in s.nodes}
    g = plan.graph
    for n in g.nodes.values():
        if n.kind == "arith":
            assert n.id in covered


EXPECT = {  # config -> (kernel kinds, count_flops, bytes_moved)
    "C1": (["gemm"], 33_554_432, 786_432),
    "C2": (["gemm"], 2_147_483_648, 12_582_912),
    "C3": (["conv"], 1_849_688_064, 13_459_456),
    "C4": (["gemm"], 34_410_070_016, 100_679_680),
    "C5": (["gemm"], 8_796_093_022_208, 3_221_225_472),
}


@pytest.mark.parametrize("name", sorted(EXPECT))
def test_config_plans_and_analytics(name):
    kinds, flops, nbytes = EXPECT[name]
    gj = common.graph_json(common.config(name)["graph"])
    k = backend.compile_graph(gj)
    assert [s.kind for s in k.plan.steps] == kinds
    assert k.flops == flops
    assert k.dfg_bytes_moved == nbytes
    assert k.scratch_bytes == 0          # fused: no intermediate materialized


def test_c4_epilogue_is_fused():
    k = backend.compile_graph(common.graph_json(common.config("C4")["graph"]))
    st = k.plan.steps[0]
    assert len(st.epi) == 3                      # contraction, +bias, relu
    assert st.epi[1].combine == 0 and st.epi[1].operand is not None
    assert st.epi[2].post == 1
    assert st.params["epi_strides"][1]["operand"] == (0, 0, 1, 0)   # bias[n] broadcast


def test_c2_plan_is_exact_semiring():
    k = backend.compile_graph(common.graph_json(common.config("C2")["graph"]))
    p = k.plan.steps[0].params
    assert (p["combine_name"], p["reduce_name"], p["beta_in_loop"]) == ("add", "max", 0)


def test_conv_guarded_form_maps_padding():
    k = backend.compile_graph(common.graph_json(common.config("C3")["graph_guarded"]))
    p = k.plan.steps[0].params
    assert (p["pad_h"], p["pad_w"], p["H"], p["W"], p["fill"]) == (1, 1, 56, 56, 0.0)
    k = backend.compile_graph(common.graph_json(common.config("C3")["graph"]))
    p = k.plan.steps[0].params
    assert (p["pad_h"], p["H"]) == (0, 58)


def test_beta_placement():
    from paper_2205_00618_b200.planner import Planner
    bp = Planner._beta_plan
    assert bp("add", "max", 0.5) == ("max", False, 0.5)
    assert bp("add", "max", -2.0) == ("min", False, -2.0)     # monotone decreasing scale
    assert bp("add", "max", 0.0) == ("max", True, 1.0)        # exact only per term
    assert bp("mul", "mul", 0.5) == ("mul", True, 1.0)
    assert bp("mul", "add", 1.0) == ("add", False, 1.0)


def test_bad_json_raises():
    with pytest.raises(GraphError):
        Graph.from_json({"vars": [], "nodes": [{"id": 0}]})


def test_compile_single_operand_contract():
    case = next(c for c in IDX["cases"] if c["name"] == "acc_transpose")
    k = backend.compile_single_operand(common.graph_json(case["graph"]))
    assert k.plan.steps[0].kind == "nest"
    with pytest.raises(backend.HasReduction):
        backend.compile_single_operand(common.graph_json(common.config("C1")["graph"]))


def test_disassemble_lists_launches():
    k = backend.compile_graph(common.graph_json(IDX["cases"][7]["graph"]))   # mlp3
    text = k.disassemble()
    assert text.count("launch.") == len(k.plan.steps)


# ---------------------------------------------------------------- live reference (dev container only)

ref = pytest.mark.skipif(not HAVE_REF, reason="reference not mounted")


def _ls():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    import loopsmith
    return loopsmith


@ref
def test_mirror_from_live_dfg_equals_json_mirror():
    ls = _ls()
    from loopsmith import serialize
    for case in IDX["cases"][:30] + IDX["configs"]:
        dfg = serialize.loads(common.graph_json(case["graph"]))
        a = plan_graph(Graph.from_dfg(dfg)).describe()
        b = plan_graph(common.graph_json(case["graph"])).describe()
        assert a == b, case["name"]
        assert Graph.from_dfg(dfg).count_flops() == ls.count_flops(dfg)
        assert Graph.from_dfg(dfg).bytes_moved() == ls.bytes_moved(dfg)


@ref
def test_compile_tree_accepts_reference_loop_tree():
    ls = _ls()
    g = ls.matmul_graph(64, 32, 48)
    k = backend.compile_tree(ls.lower(g), ls.avx512_like())
    assert k.flops == ls.count_flops(g)
    assert k.slot_shapes == {0: (64, 32), 1: (32, 48), 2: (64, 48)}
    assert k.program.lanes == 16


@ref
def test_errors_are_reference_classes():
    ls = _ls()
    assert issubclass(backend.BlockTooLarge, ls.BlockTooLarge)
    assert issubclass(backend.HasReduction, ls.HasReduction)
    assert issubclass(backend.ShapeMismatch, ls.ShapeMismatch)


@ref
def test_install_rebinds_reference_modules():
    ls = _ls()
    import loopsmith.backend
    import loopsmith.session  # noqa: F401
    import paper_2205_00618_b200 as P
    orig = loopsmith.backend.execute
    done = P.install()
    try:
        for name in ("loopsmith.backend.execute", "loopsmith.session.compile_tree",
                     "loopsmith.tuner.execute", "loopsmith.cli.compile_tree"):
            assert name in done
        assert ls.compile_tree is backend.compile_tree
        assert loopsmith.backend.execute is backend.execute   # feedback.benchmark's lazy import
    finally:
        P.uninstall()
    assert loopsmith.backend.execute is orig


def test_disassemble_renders_balanced_loop_nests():
    # reference cli.py:56-72 / session.py:247-250 callers look for loop.begin/loop.end
    for case in IDX["cases"]:
        k = backend.compile_graph(common.graph_json(case["graph"]))
        text = k.disassemble()
        assert text.count("loop.begin") == text.count("loop.end") >= len(k.plan.steps), case["name"]


def test_modeled_memory_counters():
    """Contractions count the schedule as register-blocked 16-B vector code
    (schedule.schedule_counters): C1's 4 x 64 block -> per k step of each of
    the 64 x 4 blocks, 16 vector loads of B and 4 broadcasts of A."""
    from paper_2205_00618_b200 import schedule
    k = backend.compile_graph(common.graph_json(common.config("C1")["graph"]))
    (st,) = k.plan.steps
    sm = st.params["schedule"]
    assert (sm.m_block, sm.n_block) == (4, 64)
    M = N = K = 256
    ld, bc, sv = schedule.schedule_counters(sm, M, N, K)
    assert ld == (M // 4) * (N // 64) * K * 16 and bc == (M // 4) * (N // 64) * K * 4 and sv == M * N // 4
    k._count(1)
    assert k.memory_access_count() == ld + bc + sv
    assert k.counters["launches"] == 1 and k.counters["loop"] == 1
