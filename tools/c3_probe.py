"""C3 conv launch-time probe: per-kernel event timing of each conv kernel,
back-to-back launches (no graph) and graph replays, with and without an L2
flush in between.  python tools/c3_probe.py [algo ...]
algo: tf32x3_nhwc | tf32x3_planar | planar_plain (LSB_CP_DBG=512: no
cooperative attribute)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2205_00618_b200 import backend, native  # noqa: E402

native.init(0)
algos = sys.argv[1:] or ["tf32x3_nhwc", "tf32x3_planar", "planar_plain"]
graph = bench.load_graph("C3")
host = bench.make_inputs("C3")
k = backend.compile_graph(graph)
dev = torch.device("cuda", 0)
tens = {}
for slot, shape in k.slot_shapes.items():
    tens[slot] = (torch.from_numpy(host[slot]).to(dev) if slot in host
                  else torch.zeros(shape, dtype=torch.float32, device=dev))
ptrs = {s: t.data_ptr() for s, t in tens.items()}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream()
for algo in algos:
    dbg = "512" if algo == "planar_plain" else algo.split("=")[1] if algo.startswith("planar_dbg=") else None
    native.setenv("LSB_CP_DBG", dbg)
    native.setenv("LSB_GEMM_ALGO", "tf32x3_planar" if dbg else algo)
    for _ in range(5):
        backend.run_device(k, ptrs, st.cuda_stream)
    torch.cuda.synchronize()
    for fl in ((False, True) if len(algos) < 4 else (True,)):
        ts = []
        for i in range(30):
            if fl:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            backend.run_device(k, ptrs, st.cuda_stream)
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
        # 20 launches back to back between two events (pipelined)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(20):
            backend.run_device(k, ptrs, st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        print(f"{algo:14s} flush={fl!s:5s} per-launch med {t[len(t) // 2]:7.2f} min {t[0]:7.2f} us | "
              f"20 back-to-back {a.elapsed_time(b) * 1e3 / 20:7.2f} us/launch", flush=True)
native.setenv("LSB_GEMM_ALGO", None)
native.setenv("LSB_CP_DBG", None)

# effective SM clock: torch.cuda._sleep spins for a number of clock64 cycles
for cyc in (20_000, 200_000, 2_000_000):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        a.record(st)
        torch.cuda._sleep(cyc)
        b.record(st)
        torch.cuda.synchronize()
    print(f"sleep {cyc} cycles: {a.elapsed_time(b) * 1e3:.2f} us -> {cyc / (a.elapsed_time(b) * 1e3):.0f} MHz")
