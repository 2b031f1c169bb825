"""C4 (4096x1024x4096 + bias + ReLU) step timing: warm L2 vs flushed L2, and
the main kernel alone (lsb_profile)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2205_00618_b200 import backend, native  # noqa: E402
import common  # noqa: E402
native.init(0)
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
k = backend.compile_graph(common.graph_json(f"graphs/{name}.json"))
bufs = common.config_inputs(name)
t = {s: torch.from_numpy(a).cuda() for s, a in bufs.items()}
for s, shape in k.slot_shapes.items():
    if s not in t:
        t[s] = torch.zeros(shape, device="cuda")
ptrs = {s: v.data_ptr() for s, v in t.items()}
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
for _ in range(3):
    backend.run_device(k, ptrs, s)
torch.cuda.synchronize()
for fl in (False, True):
    ts, ks = [], []
    for _ in range(5):
        if fl:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        native.profile(True)
        e0.record()
        backend.run_device(k, ptrs, s)
        e1.record()
        torch.cuda.synchronize()
        ks.append(native.last_kernel_ms())
        native.profile(False)
        ts.append(e0.elapsed_time(e1))
    print(f"{name} flush={fl}: step ms {min(ts):.4f} (mean {sum(ts)/len(ts):.4f})  main kernel ms {min(ks):.4f}")
