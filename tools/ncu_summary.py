"""Summarise an ncu --set full report into profiles/ (run here, no GPU).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_xxx.json [--traffic-key NAME]

Writes the headline metrics (duration, DRAM bytes, pipe utilisation, stall
reasons) and, with --traffic-key, records dram read+write bytes per launch in
profiles/traffic.json (read by bench.py for roofline.traffic).
"""

import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    if rep.endswith(".csv"):   # an `ncu -i ... --page raw --csv` export
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    res = {"report": os.path.basename(rep), "kernel": d.get("Kernel Name", ("", ""))[0]}
    for k in KEYS:
        if k in d:
            v, u = d[k]
            try:
                res[k] = float(v.replace(",", ""))
                res[k + ".unit"] = u
            except ValueError:
                res[k] = v
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
              for h, (v, _) in d.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    res["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}

    def bytes_of(k):
        v, u = d[k]
        return float(v.replace(",", "")) * SCALE.get(u, 1)

    if "dram__bytes_read.sum" in d:
        res["dram_bytes_per_launch"] = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))
    if key and "dram_bytes_per_launch" in res:
        tp = os.path.join(os.path.dirname(out), "traffic.json")
        t = json.load(open(tp)) if os.path.exists(tp) else {}
        t[key] = {"dram_bytes_per_launch": res["dram_bytes_per_launch"], "source": os.path.basename(out)}
        json.dump(t, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
