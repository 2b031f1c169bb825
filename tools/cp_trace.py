"""Summarise a conv_planar trace (LSB_CONV_TRACE=path): per-CTA globaltimer
stamps relative to the earliest start, in microseconds.
slots: 0 start, 1-15 MMA job ends, 16-30 converter job arrivals, 31-45
epilogue chunk folds, 46 publish, 47+4s wait start, 48+4s wait end,
49+4s store end (segment s), 63 exit."""
import sys

import numpy as np

rows, srows = [], []
with open(sys.argv[1]) as f:
    head = f.readline()
    for line in f:
        if line.startswith("S "):
            srows.append([int(x) for x in line.split()[1:]])
        else:
            rows.append([int(x) for x in line.split()])
a = np.array(rows, dtype=np.float64)
g0, g1 = a[:, 62].copy(), a[:, 61].copy()
if (g0 > 0).all():
    t0 = g0.min()
    print("globaltimer (us): CTA start min %.2f max %.2f | end min %.2f med %.2f max %.2f" % (
        0.0, (g0.max() - t0) / 1e3, (g1.min() - t0) / 1e3, (np.median(g1) - t0) / 1e3, (g1.max() - t0) / 1e3))
# clock64 stamps: per-CTA cycles from its own start, shown in k-cycles
a = np.where(a > 0, (a - a[:, :1]) / 1e3, np.nan)
print(head.strip())
print("start  min %.2f max %.2f us" % (np.nanmin(a[:, 0]), np.nanmax(a[:, 0])))
print("exit   min %.2f med %.2f max %.2f us" % (np.nanmin(a[:, 63]), np.nanmedian(a[:, 63]), np.nanmax(a[:, 63])))
for b in list(range(0, 4)) + [int(np.nanargmax(a[:, 63]))]:
    r = a[b]
    f = lambda sl: " ".join("%.1f" % x for x in r[sl] if not np.isnan(x))
    print(f"cta {b}: start {r[0]:.2f} | conv {f(slice(16, 31))} | mma {f(slice(1, 16))} | fold {f(slice(31, 46))}"
          f" | pub {r[46]:.2f} | seg(wait0,wait1,store) {f(slice(47, 59))} | exit {r[63]:.2f}")
if srows:
    sa = np.array(srows, dtype=np.float64)
    for b in (0, 1):
        pre, post = sa[b, 0::2], sa[b, 1::2]
        m = post > 0
        base = pre[m][0]
        print(f"cta {b} stage clocks (cycles from first): wait-start", " ".join("%d" % (x - base) for x in pre[m]))
        print(f"cta {b}                                    waited    ", " ".join("%d" % x for x in (post - pre)[m]))
        jb = sa[b, 100:127].reshape(9, 3)
        print(f"cta {b} job starts (halo wait, c_empty wait, go):", "; ".join(
            "%d %d %d" % tuple(x - base for x in r) for r in jb if r[0] > 0))
