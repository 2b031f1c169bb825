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
a = a[a[:, 62] > 0] if (a[:, 62] > 0).any() else a     # CTAs that ran
a_raw = a.copy()
g0, g1 = a[:, 62].copy(), a[:, 61].copy()
if (a[:, 60] > 0).all():
    ent, st0, ex = a[:, 60], a[:, 0], a[:, 63]
    mhz = (ex - ent) / (g1 - g0) * 1e3
    print("entry->start(slot 0) cycles: min %d med %d max %d | entry->exit cycles med %d | SM clock %.0f MHz (med)" % (
        (st0 - ent).min(), np.median(st0 - ent), (st0 - ent).max(), np.median(ex - ent), np.median(mhz)))
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
          f" | raw-in {f(slice(50, 56))} | mma-go {f(slice(56, 60))} | store-end {r[49]:.2f} | exit {r[63]:.2f}")
if srows:
    sa = np.array(srows, dtype=np.float64)
    for b in (0, 1):
        base = a_raw[b, 0]
        for job in range(4):
            cells = []
            for w in range(4):
                ev = sa[b, 32 * job + 8 * w: 32 * job + 8 * w + 4]
                cells.append("/".join("%.2f" % ((x - base) / 1e3) if x > 0 else "-" for x in ev))
            print(f"cta {b} job {job} converter warps (raw-in/halo-free/converted/bar, k-cycles):", "  ".join(cells))
            m = sa[b, 32 * job + 4: 32 * job + 7]
            if job == 3:
                print(f"cta {b} epilogue tail (stores start):", "%.2f" % ((sa[b, 124] - base) / 1e3))
            print(f"cta {b} job {job} mma warp (start, halo_full passed, c_empty passed):",
                  " ".join("%.2f" % ((x - base) / 1e3) for x in m))
