"""Per-call time of forced tensor-core GEMMs (resized semiring_mul_add graph)
for a few shapes, run_device with device-resident operands."""
import os, sys
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tests")]
from test_gpu_edges import _graph
from paper_2205_00618_b200 import backend, native
native.init(0)
native.setenv("LSB_GEMM_ALGO", "tf32x3")
st = torch.cuda.current_stream()
for (m, k, n) in [(4096, 1024, 4096), (4096, 4096, 4096), (8192, 1024, 8192), (4096, 16384, 4096)]:
    kern = backend.compile_graph(_graph("semiring_mul_add", m=m, k=k, n=n))
    tens = {s: torch.randn(shp, device="cuda") for s, shp in kern.slot_shapes.items()}
    ptrs = {s: t.data_ptr() for s, t in tens.items()}
    for _ in range(3): backend.run_device(kern, ptrs, st.cuda_stream)
    torch.cuda.synchronize()
    native.profile(True)
    backend.run_device(kern, ptrs, st.cuda_stream)
    torch.cuda.synchronize()
    kms = round(native.last_kernel_ms() * 1e3, 1)
    native.profile(False)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10): backend.run_device(kern, ptrs, st.cuda_stream)
    b.record(st); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 10
    print((m, k, n), "%.1f us/call  %.1f TF/s" % (t * 1e3, 2 * m * n * k / (t * 1e-3) / 1e12), "kernel", kms, flush=True)
