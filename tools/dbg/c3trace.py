"""Traced planar conv launches at C3 (each launch syncs to dump its trace)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2205_00618_b200 import backend, native
native.init(0)
k = backend.compile_graph(bench.load_graph("C3"))
host = bench.make_inputs("C3")
dev = torch.device("cuda", 0)
tens = {s: (torch.from_numpy(host[s]).to(dev) if s in host else torch.zeros(sh, device=dev)) for s, sh in k.slot_shapes.items()}
ptrs = {s: t.data_ptr() for s, t in tens.items()}
native.setenv("LSB_GEMM_ALGO", "tf32x3_planar")
for i in range(5):
    backend.run_device(k, ptrs, 0)
torch.cuda.synchronize()
native.setenv("LSB_CONV_TRACE", sys.argv[1])
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    torch.cuda._sleep(2_000_000)   # keep the clock up between traced launches
    backend.run_device(k, ptrs, 0)
torch.cuda.synchronize()
