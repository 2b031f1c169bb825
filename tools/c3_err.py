"""C3 accuracy headroom: max |got - ref| / (atol + rtol |ref|) on image 0 (1.0 = at the tolerance)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2205_00618_b200 import backend, native  # noqa: E402
import common  # noqa: E402
native.init(0)
cfg = common.config("C3")
bufs = common.config_inputs("C3")
k = backend.compile_graph(common.graph_json(cfg["graph"]))
out = np.zeros(8 * 64 * 56 * 56, np.float32)
ins = {s: a for s, a in bufs.items() if s != 2}
ins[2] = out
backend.execute(k, ins)
o = out.reshape(8, 64, 56, 56)[0].astype(np.float64)
d = np.load(common.GOLDEN + "/" + cfg["data"])
ref = d["ref_img0"].astype(np.float64).reshape(64, 56, 56)
r = np.abs(o - ref) / (common.ATOL + common.RTOL * np.abs(ref))
print("C3 headroom max %.4f  mean %.5f  max_abs_err %.3e  max|ref| %.2f" % (r.max(), r.mean(), np.abs(o - ref).max(), np.abs(ref).max()))
