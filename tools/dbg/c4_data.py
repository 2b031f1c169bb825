"""C4 graph (4096x1024x4096 + bias + ReLU) timed with different input distributions."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2205_00618_b200 import backend, native
native.init(0)
k = backend.compile_graph(bench.load_graph("C4"))
dev = torch.device("cuda", 0)
host = bench.make_inputs("C4")
st = torch.cuda.current_stream()
for dist in ("spec", "uniform", "normal1", "spec_x1000"):
    rng = np.random.default_rng(0)
    tens = {}
    for s, shp in k.slot_shapes.items():
        if s in host:
            a = host[s]
            if dist == "uniform" and a.ndim == 2: a = rng.uniform(-1, 1, a.shape).astype(np.float32)
            if dist == "normal1" and a.ndim == 2: a = rng.standard_normal(a.shape).astype(np.float32)
            if dist == "spec_x1000" and a.ndim == 2: a = a * 1000
            tens[s] = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        else:
            tens[s] = torch.zeros(shp, device=dev)
    ptrs = {s: t.data_ptr() for s, t in tens.items()}
    for _ in range(5): backend.run_device(k, ptrs, st.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20): backend.run_device(k, ptrs, st.cuda_stream)
    b.record(st); torch.cuda.synchronize()
    print(dist, "%.1f us per call" % (a.elapsed_time(b) * 1e3 / 20), flush=True)
