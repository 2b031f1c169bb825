"""The C ABI rejects bad descriptors with an error code and a message
(lsb_last_error) instead of launching, and empty extents are no-ops."""
import numpy as np
import pytest
import torch

from paper_2205_00618_b200 import native

pytestmark = pytest.mark.gpu


def _gemm(M=8, N=8, K=8, **kw):
    native.init(0)
    A = torch.rand(max(M, 1), max(K, 1), device="cuda")
    B = torch.rand(max(K, 1), max(N, 1), device="cuda")
    C = torch.full((max(M, 1), max(N, 1)), 7.0, device="cuda")
    d = native.GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, 1
    d.A, d.sa_m, d.sa_k = A.data_ptr(), max(K, 1), 1
    d.B, d.sb_k, d.sb_n = B.data_ptr(), max(N, 1), 1
    d.C, d.sc_m, d.sc_n = C.data_ptr(), max(N, 1), 1
    d.combine, d.reduce, d.beta = 1, 0, 1.0
    for k, v in kw.items():
        setattr(d, k, v)
    return d, (A, B, C)


@pytest.mark.parametrize("field,value,msg", [
    ("M", -1, "bad extents"), ("batch", 0, "bad extents"), ("combine", 9, "bad operator"),
    ("A", 0, "null operand"), ("n_epi", 99, ""),
])
def test_bad_gemm_desc_is_rejected(field, value, msg):
    d, keep = _gemm(**{field: value})
    with pytest.raises(native.NativeError) as e:
        native.semiring_gemm(d)
    assert msg in str(e.value)


def test_empty_rows_are_a_noop():
    d, (A, B, C) = _gemm(M=0)
    native.semiring_gemm(d)
    torch.cuda.synchronize()
    assert float(C[0, 0]) == 7.0


def test_forced_tf32x3_on_unsupported_pair_is_an_error():
    d, keep = _gemm(combine=0, reduce=2, algo=2)   # (add, max) has no tensor-core form
    with pytest.raises(native.NativeError):
        native.semiring_gemm(d)
