"""Planar conv on a list of pad-1 3x3 geometries, one subprocess each (a
fault in one does not hide the others): python planar_shapes.py n,ci,hw,co ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import numpy as np
    import common
    from test_gpu_edges import _graph, _run, _conv_pad1_f64
    from paper_2205_00618_b200 import backend, native
    native.setenv("LSB_GEMM_ALGO", "tf32x3_planar")
    n, ci, hw, co = map(int, sys.argv[2].split(","))
    gj = _graph("conv_pad1_small", n=n, ci=ci, hp=hw, wp=hw, h=hw, w=hw, co=co)
    k = backend.compile_graph(gj)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (n, ci, hw, hw)).astype(np.float32)
    w = rng.normal(0, 0.1, (co, ci, 3, 3)).astype(np.float32)
    got = _run(k, {0: x, 1: w})[2].reshape(n, co, hw, hw)
    ok = common.strict_ok(got, _conv_pad1_f64(x, w))
    print("strict", float(ok.mean()))
    sys.exit(0)
for g in sys.argv[1:]:
    r = subprocess.run([sys.executable, __file__, "one", g], capture_output=True, text=True, timeout=120)
    tail = [l for l in (r.stdout + r.stderr).splitlines() if "CUDAEvent" not in l][-1:]
    print(g, "rc", r.returncode, tail, flush=True)
