"""Forced tensor-core GEMM on small/ragged shapes vs f64, under knob variants."""
import os, sys
import numpy as np
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests")]
from test_gpu_edges import _graph, _run
from paper_2205_00618_b200 import backend, native
native.setenv("LSB_GEMM_ALGO", "tf32x3")
for env in ([], [("LSB_NO_ILV", "1")], [("LSB_SCALAR_SPLIT", "1")]):
    for k_, v_ in env: native.setenv(k_, v_)
    for (m, k, n) in [(37, 29, 53), (64, 32, 64), (128, 16, 256), (128, 64, 256), (256, 1024, 512), (37, 32, 64), (64, 29, 64), (64, 32, 53)]:
        gj = _graph("semiring_mul_add", m=m, k=k, n=n)
        kern = backend.compile_graph(gj)
        rng = np.random.default_rng(1)
        A = rng.uniform(-10, 10, (m, k)).astype(np.float32); B = rng.uniform(-10, 10, (k, n)).astype(np.float32)
        got = _run(kern, {0: A, 1: B})
        out = [s for s in got if s not in (0, 1)][0]
        g = got[out].reshape(m, n).astype(np.float64); r = A.astype(np.float64) @ B.astype(np.float64)
        d = np.abs(g - r)
        print(env, (m, k, n), "metric %.2e" % (d.max() / np.abs(r).max()), "worst at", np.unravel_index(d.argmax(), d.shape), flush=True)
    for k_, v_ in env: native.setenv(k_, None)
