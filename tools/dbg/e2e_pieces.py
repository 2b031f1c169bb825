"""C5 execute() from pinned host buffers with different blocked piece counts."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2205_00618_b200 import backend, native
native.init(0)
k = backend.compile_graph(bench.load_graph("C5"))
host = bench.make_inputs("C5")
pa, pb, pc = (native.PinnedBuffer(host[0].shape), native.PinnedBuffer(host[1].shape),
              native.PinnedBuffer((16384, 16384)))
pa.array[...] = host[0]; pb.array[...] = host[1]
bufs = {0: pa.array, 1: pb.array, 2: pc.array}
for npieces in [int(x) for x in sys.argv[1:]] or [16, 24, 32]:
    backend.BLOCK_PIECES = npieces
    backend.execute(k, bufs)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); backend.execute(k, bufs); ts.append(time.perf_counter() - t0)
    print(npieces, "pieces: %.1f ms median, %.1f TF/s" % (np.median(ts) * 1e3, 2 * 16384**3 / np.median(ts) / 1e12), flush=True)
