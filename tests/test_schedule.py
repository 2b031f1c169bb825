"""Schedule fidelity and caller compatibility (§8(f)2) of
the schedule mapping (paper_2205_00618_b200/schedule.py), on CPU.

Schedules are built with the reference frontend when it is importable (this
dev container); the GPU box has no copy of it, so these tests skip there.
Reference tests mirrored: test_lowering.py:102-121 (packed scratch),
test_feedback.py:147-164 (blocked moves less memory than naive),
test_tuner.py:42-47 (the counters give the tuner something to rank)."""
from __future__ import annotations

import pytest

ls = pytest.importorskip("loopsmith")
sch = pytest.importorskip("loopsmith.schedule")

from paper_2205_00618_b200 import backend  # noqa: E402


def _reorder(g, order):
    for node in g:
        names = [v.name for v in node.order]
        sch.apply_action(g, sch.ReorderAction(node.id, [n for n in order if n in names]
                                              + [n for n in names if n not in order]))


def _mm(m, k, n, splits=(), order=None):
    g = ls.matmul_graph(m, k, n)
    for var, f in splits:
        sch.split(g, sch.find_var(g, var), f)
    if order:
        _reorder(g, order)
    return g


def _gemm_step(kern):
    (st,) = [s for s in kern.plan.steps if s.kind == "gemm"]
    return st


def test_packed_scratch_is_8192_elements():
    """test_lowering.py:102-121 on the B200 backend: staging a k-tile of B
    under shared outer loops is a 128 x 64 packed panel = 32 KB of scratch."""
    g = _mm(512, 512, 512, [("m", 5), ("n", 64), ("k", 128)], ["n_o", "k_o", "m_o", "k_i", "m_i", "n_i"])
    read_b = g[1]
    sch.stage(g, read_b, next(v for v in read_b.order if v.name == "k_i"))
    tree = ls.lower(g)
    assert ls.alloc_size(read_b, tree) == 8192
    kernel = backend.compile_tree(tree, ls.avx512_like())
    assert kernel.scratch_bytes >= 8192 * 4
    st = _gemm_step(kernel)
    assert st.params["schedule"].staged, "the staged Read is recorded on the launch"
    assert "staged panel" in kernel.program.disassemble()


def test_blocked_mm_moves_less_memory_than_naive():
    """test_feedback.py:147-164: the blocked schedule's modeled memory
    accesses are far below the naive schedule's (the tuner's score)."""
    naive = backend.compile_tree(ls.lower(_mm(256, 256, 256)), ls.avx512_like())
    blocked = backend.compile_tree(
        ls.lower(_mm(256, 256, 256, [("m", 4), ("n", 64)], ["m_o", "n_o", "k", "m_i", "n_i"])),
        ls.avx512_like())
    naive._count(1)
    blocked._count(1)
    assert blocked.memory_access_count() * 2 < naive.memory_access_count()


def test_schedules_select_launch_configurations():
    """Different schedules of the same contraction select different tiles:
    a small register block -> 64-row SIMT / 128-wide 3xTF32 tiles, a 4 x 64
    block -> the default tiles, an outermost reduction loop -> split-K."""
    naive = _gemm_step(backend.compile_tree(ls.lower(_mm(2048, 2048, 2048)), ls.avx512_like()))
    assert naive.params["tile_m"] == 64 and naive.params["tile_n"] == 128
    blocked = _gemm_step(backend.compile_tree(
        ls.lower(_mm(2048, 2048, 2048, [("m", 4), ("n", 64)], ["m_o", "n_o", "k", "m_i", "n_i"])),
        ls.avx512_like()))
    assert blocked.params["tile_m"] == 0 and blocked.params["tile_n"] == 0 and blocked.params["split_k"] == 0
    ksplit = _gemm_step(backend.compile_tree(
        ls.lower(_mm(256, 4096, 256, [("k", 512), ("m", 4), ("n", 64)], ["k_o", "m_o", "n_o", "k_i", "m_i", "n_i"])),
        ls.avx512_like()))
    assert ksplit.params["split_k"] == 8
    assert "split-K 8" in backend.compile_tree(
        ls.lower(_mm(256, 4096, 256, [("k", 512), ("m", 4), ("n", 64)], ["k_o", "m_o", "n_o", "k_i", "m_i", "n_i"])),
        ls.avx512_like()).program.disassemble()


def test_counters_follow_the_register_block():
    """Counters shrink as the register block grows (what tune ranks by)."""
    def count(splits, order):
        k = backend.compile_tree(ls.lower(_mm(64, 64, 64, splits, order)), ls.avx512_like())
        k._count(1)
        return k.memory_access_count()
    naive = count((), None)
    row = count([("n", 16)], ["m", "n_o", "k", "n_i"])
    block = count([("m", 4), ("n", 64)], ["m_o", "n_o", "k", "m_i", "n_i"])
    assert naive > row > block and block * 2 < naive
