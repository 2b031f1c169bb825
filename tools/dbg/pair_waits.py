"""MMA-warp filter waits per tap pair from a conv_planar trace (S rows, slots 8 + 4i / 9 + 4i)."""
import sys
import numpy as np
S = np.array([l.split()[1:] for l in open(sys.argv[1]) if l.startswith("S")], dtype=np.int64)
R = np.array([l.split() for l in open(sys.argv[1]) if not l.startswith(("#", "S"))], dtype=np.int64)
for b in (0, 1, 2):
    base = R[b, 0]
    pre, post = S[b, 8:104:4], S[b, 9:105:4]
    m = post > 0
    print(f"cta {b} pair wait start (k-cycles):", " ".join("%.2f" % ((x - base) / 1e3) for x in pre[m]))
    print(f"cta {b} waited (cycles):         ", " ".join("%d" % x for x in (post - pre)[m]))
    print(f"cta {b} mma-go:", " ".join("%.2f" % ((R[b, 56 + i] - base) / 1e3) for i in range(4)),
          "| mma job end:", " ".join("%.2f" % ((R[b, 1 + i] - base) / 1e3) for i in range(4)))
