"""Time the C3 conv through the C ABI: eager (host overhead included) and
CUDA-graph replay (device time), plus LSB profile of the conv kernel alone."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2205_00618_b200 import backend, native  # noqa: E402
import common  # noqa: E402
native.init(0)
k = backend.compile_graph(common.graph_json("graphs/C3g.json"))
bufs = common.config_inputs("C3g")
t = {s: torch.from_numpy(a).cuda() for s, a in bufs.items()}
t[2] = torch.empty(8, 64, 56, 56, device="cuda")
ptrs = {s: v.data_ptr() for s, v in t.items()}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    backend.run_device(k, ptrs, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    backend.run_device(k, ptrs, s)
e1.record()
torch.cuda.synchronize()
print("conv ms (eager, host-bound)", e0.elapsed_time(e1) / 20)
if reps > 1 and not os.environ.get("LSB_CONV_TRACE"):
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(20):
                backend.run_device(k, ptrs, side.cuda_stream)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print("conv ms (graph)", e0.elapsed_time(e1) / 20)
    native.profile(True)
    backend.run_device(k, ptrs, s)
    torch.cuda.synchronize()
    print("conv kernel ms (profile)", native.last_kernel_ms())
    native.profile(False)
