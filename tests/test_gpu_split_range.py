"""Range of the fp16 hi/lo split (tf32x3_gemm.cuh): operands are scaled by a
power of two per A row and per 128-column block of B before the split, and
the accumulator is unscaled in the epilogue.  Rows and column blocks whose
magnitudes differ by up to 1e+-30, zero rows and blocks, fp32 subnormals and
mixed scales inside one row must all land within the strict rule of their
own scale (checked on C / (row scale x column scale) against f64)."""

import numpy as np
import pytest

import common
from test_gpu_edges import _graph, _run

pytestmark = pytest.mark.gpu


def _check(got, A, B, rs, cs):
    """Strict rule on the natural scale for short K; for K >= 1024 uniform
    data fails it on a few near-zero outputs with any fp32 accumulation (the
    VM's too, test_tf32x3_tail_split), so the reference metric plus a
    >= 99.9 % strict fraction there."""
    ref = A.astype(np.float64) @ B.astype(np.float64)
    scale = np.outer(rs, cs)
    g = got.astype(np.float64) / scale
    r = ref / scale
    ok = common.strict_ok(g, r)
    if A.shape[1] < 1024:
        assert ok.all(), (float(ok.mean()), common.ref_metric(g, r))
    else:
        assert common.ref_metric(g, r) <= 1e-4 and ok.mean() >= 0.999, (float(ok.mean()), common.ref_metric(g, r))


@pytest.mark.parametrize("m,k,n", [(300, 200, 520), (1024, 1024, 1024)])
def test_split_row_and_block_scales(m, k, n, monkeypatch):
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    rng = np.random.default_rng(m + k + n)
    rs = 10.0 ** rng.integers(-15, 16, m)                    # per-row magnitude
    cs = 10.0 ** rng.integers(-15, 16, (n + 127) // 128)     # per 128-column block
    cs = np.repeat(cs, 128)[:n]
    A = (rng.uniform(-1, 1, (m, k)) * rs[:, None]).astype(np.float32)
    B = (rng.uniform(-1, 1, (k, n)) * cs[None, :]).astype(np.float32)
    A[5] = 0.0                                   # a zero row
    B[:, 128:256] = 0.0 if n > 256 else B[:, 128:256]   # a zero block
    kern = __import__("paper_2205_00618_b200.backend", fromlist=["x"]).compile_graph(
        _graph("semiring_mul_add", m=m, k=k, n=n))
    got = _run(kern, {0: A, 1: B})
    out = [s for s in got if s not in (0, 1)][0]
    c = got[out].reshape(m, n)
    rs2, cs2 = rs.copy(), cs.copy()
    rs2[5] = 1.0
    if n > 256:
        cs2[128:256] = 1.0
    _check(c, A, B, rs2, cs2)


def test_split_mixed_scales_in_a_row(monkeypatch):
    """Within one row, values 1e-6 .. 1e6 apart: the small ones lose low bits
    as fp16 subnormals after the row's scaling; the result stays inside the
    strict rule relative to the row's natural scale."""
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    m, k, n = 256, 512, 384
    rng = np.random.default_rng(11)
    A = (rng.uniform(-1, 1, (m, k)) * 10.0 ** rng.integers(-6, 7, (m, k))).astype(np.float32)
    B = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    kern = __import__("paper_2205_00618_b200.backend", fromlist=["x"]).compile_graph(
        _graph("semiring_mul_add", m=m, k=k, n=n))
    got = _run(kern, {0: A, 1: B})
    out = [s for s in got if s not in (0, 1)][0]
    ref = A.astype(np.float64) @ B.astype(np.float64)
    # per-element tolerance on the row's own scale: 1e-4 of sum |a||b| (the
    # VM's fp32 accumulation sits at ~K x 2^-24 of it)
    bound = 1e-5 * (np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64))
    d = np.abs(got[out].reshape(m, n).astype(np.float64) - ref)
    assert (d <= 1e-5 + bound).all(), float((d / (1e-5 + bound)).max())


def test_split_subnormal_operands(monkeypatch):
    """fp32 subnormal inputs (|x| < 2^-126) scale up into fp16's range."""
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3")
    m, k, n = 128, 256, 256
    rng = np.random.default_rng(12)
    A = (rng.uniform(-1, 1, (m, k)) * 1e-39).astype(np.float32)
    B = (rng.uniform(-1, 1, (k, n)) * 1e30).astype(np.float32)
    kern = __import__("paper_2205_00618_b200.backend", fromlist=["x"]).compile_graph(
        _graph("semiring_mul_add", m=m, k=k, n=n))
    got = _run(kern, {0: A, 1: B})
    out = [s for s in got if s not in (0, 1)][0]
    _check(got[out].reshape(m, n), A, B, np.full(m, 1e-39), np.full(n, 1e30))
