"""Per-kernel SASS instruction counts of liblsb.so (cuobjdump -sass, run here:
no GPU needed) -- the evidence that the kernels use tcgen05 (UTCHMMA, UTCBAR,
LDTM), TMA (UTMALDG / UTMASTG / UBLKCP) and the paired FP32 ops (FFMA2,
FADD2, FMNMX3).  python tools/sass_counts.py > profiles/r02_sass_counts.json"""
import collections
import json
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2205_00618_b200/liblsb.so"
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "ELECT", "FFMA2", "FFMA", "FADD2",
        "FMNMX3", "FMNMX", "FADD", "LDS", "STS", "LDG", "STG", "LDGSTS", "SHFL", "RED", "ATOMG", "BAR"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if kern and m:
        op = m.group(2)
        counts[kern][op] += 1
        counts[kern]["_total"] += 1
res = {}
for k, c in counts.items():
    demangled = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    short = re.sub(r"\(.*", "", demangled)
    ent = {"instructions": c["_total"], **{key: c[key] for key in KEYS if c[key]}}
    res.setdefault(short, []).append({"mangled": k, **ent})
print(json.dumps(res, indent=1))
