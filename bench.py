#!/usr/bin/env python
"""Benchmark of the B200 loop-nest backend (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl b200|reference]

Metric: GFLOP/s per contraction config and fraction of the B200 FP32
roofline.  The headline line is the sharded config C5 (fp32 GEMM 16384^3,
rows of A/C split across the N ranks, B replicated, no data-path collective);
at N=1 the other configs C1..C4 are measured too and reported under
"per_config".  A "step" is one pass of the hot path over one batch of the
synthetic input (one full contraction).

value      device time (CUDA events on the launching stream, max over ranks),
           inputs resident in HBM; whole-job GFLOP/s = total flops / time.
e2e        the same contraction through the public drop-in API
           (backend.execute) from pinned host buffers: H2D of the inputs, the
           kernels and D2H of the result inside the timed region.
roofline   dominant kernel's achieved TFLOP/s (algorithmic 2*M*N*K / its own
           average launch duration, CUDA events placed by liblsb around that
           launch).  3xTF32 tensor-core path: against measured bf16 sustained
           / 2 (tf32) / 3 (passes); SIMT path: against the FP32 peak
           148 SMs x 128 lanes x 2 flop x 1965 MHz = 74.4 TFLOP/s (computed
           from MEASURED_PEAKS.json sm_max_mhz; no measured FP32 peak exists).
cpu_baseline  oracle/vmport.c (C restatement of the reference VM arithmetic,
           bit-exact with it) on a bounded row sample, all host threads.
--impl reference   times that same CPU path as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP32_LANES_PER_SM = 128

CONFIGS = {
    "C1": dict(kind="gemm", M=256, N=256, K=256, combine="mul", reduce="add",
               desc="fp32 GEMM 256^3 (seed 0, U[-1,1))"),
    "C2": dict(kind="gemm", M=1024, N=1024, K=1024, combine="add", reduce="max",
               desc="max-plus 1024^3 (seed 1, U[-10,10)), bit-exact"),
    "C3": dict(kind="conv", desc="conv NCHW 8x64x56x56 -> 64, 3x3, pad 1 (seed 2)"),
    "C4": dict(kind="gemm", M=4096, N=4096, K=1024, combine="mul", reduce="add",
               desc="MLP ReLU(X.W+b) 4096x1024x4096, bias+ReLU fused (seed 3)"),
    "C5": dict(kind="gemm", M=16384, N=16384, K=16384, combine="mul", reduce="add",
               desc="fp32 GEMM 16384^3 (seed 4, U[-1,1)), rows sharded over ranks"),
}
FLOPS = {"C1": 2 * 256 ** 3, "C2": 2 * 1024 ** 3, "C3": 2 * 8 * 64 * 56 * 56 * 64 * 9,
         "C4": 2 * 4096 * 1024 * 4096 + 2 * 4096 * 4096, "C5": 2 * 16384 ** 3}
GRAPH = {"C1": "C1", "C2": "C2", "C3": "C3g", "C4": "C4", "C5": "C5"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------- graphs / inputs

def load_graph(name: str, rows: int | None = None) -> dict:
    with open(os.path.join(ROOT, "tests", "golden", "graphs", f"{GRAPH[name]}.json")) as f:
        obj = json.load(f)
    if rows is not None:
        # shard: the same graph with the M var (and its split lineage) resized
        byid = {v["id"]: v for v in obj["vars"]}
        m = next(v for v in obj["vars"] if v["name"] == "m" and v["origin"] is None)
        m["size"] = rows
        for v in obj["vars"]:
            o = v["origin"]
            if o is not None and o["parent"] == m["id"]:
                f = o["factor"]
                v["size"] = f if o["part"] == "inner" else -(-rows // f)
        del byid
    return obj


def make_inputs(name: str, r0: int = 0, r1: int | None = None) -> dict:
    """Seeded inputs of SURVEY §8(d); for C5 only rows [r0, r1) of A."""
    if name == "C5":
        rng = np.random.default_rng(4)
        n = 16384
        # draw A row-block by row-block so a shard never holds all of A
        A = None
        step = 1024
        for lo in range(0, n, step):
            blk = rng.uniform(-1, 1, (step, n)).astype(np.float32)
            if r1 is not None and (lo + step <= r0 or lo >= r1):
                continue
            a, b = max(r0, lo), min(r1 if r1 is not None else n, lo + step)
            part = blk[a - lo:b - lo]
            A = part if A is None else np.concatenate([A, part])
        B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        return {0: A, 1: B}
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import common
    if name == "C3":
        return common.config_inputs("C3g")
    return common.config_inputs(name)


# ---------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU path

def cpu_time(name: str, budget_s: float = 8.0) -> dict:
    """oracle/vmport.c (the reference VM's arithmetic, bit-exact) on all host
    threads, on a bounded row sample of the config; GFLOP/s extrapolated by
    flops of the sample / time."""
    from oracle import vmport
    cfg = CONFIGS[name]
    threads = vmport.cores()
    if name == "C3":
        bufs = make_inputs("C3")
        t0 = time.perf_counter()
        imgs = 0
        while imgs < 8 and (imgs == 0 or time.perf_counter() - t0 < budget_s):
            vmport.conv2d(bufs[0], bufs[1], pad=1, images=(imgs, imgs + 1), threads=threads)
            imgs += 1
        dt = time.perf_counter() - t0
        flops = FLOPS["C3"] * imgs / 8
        sample = f"{imgs} of 8 images"
    else:
        if name == "C5":
            bufs = make_inputs("C5", 0, 64)
        else:
            bufs = make_inputs(name)
        A, B = bufs[0], bufs[1]
        kw = {}
        if name == "C4":
            kw = dict(bias=bufs[2], post="relu")
        M = A.shape[0]
        rows = 0
        blk = max(threads * 4, 8)
        out = np.zeros((M, B.shape[1]), np.float32)
        t0 = time.perf_counter()
        while rows < M and (rows == 0 or time.perf_counter() - t0 < budget_s):
            r1 = min(M, rows + blk)
            vmport.gemm(A, B, cfg["combine"], cfg["reduce"], rows=(rows, r1), out=out,
                        threads=threads, **kw)
            rows = r1
        dt = time.perf_counter() - t0
        total_rows = cfg["M"]
        flops = FLOPS[name] * rows / total_rows
        sample = f"{rows} of {total_rows} output rows"
    return {"value": flops / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"{name}: {sample} in {dt:.2f}s (oracle/vmport.c, VM f32 arithmetic)"}


# ---------------------------------------------------------------- GPU arm

def gpu_config_run(name: str, steps: int, warmup: int, torch, rank: int, world: int,
                   flush_l2: bool, want_e2e: bool):
    from paper_2205_00618_b200 import backend, native
    cfg = CONFIGS[name]
    if name == "C5":
        rows = cfg["M"] // world
        r0 = rank * rows
        graph = load_graph("C5", rows=rows)
        host = make_inputs("C5", r0, r0 + rows)
    else:
        graph = load_graph(name)
        host = make_inputs(name)
    k = backend.compile_graph(graph)
    dev = torch.device("cuda", torch.cuda.current_device())
    tens = {}
    for slot, shape in k.slot_shapes.items():
        if slot in host:
            tens[slot] = torch.from_numpy(np.ascontiguousarray(host[slot])).to(dev)
        else:
            tens[slot] = torch.zeros(shape, dtype=torch.float32, device=dev)
    ptrs = {s: t.data_ptr() for s, t in tens.items()}
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if flush_l2 else None

    for _ in range(warmup):
        backend.run_device(k, ptrs, sh)
    torch.cuda.synchronize()
    # one step = the plan's launches, captured once as a CUDA graph so host
    # launch latency never sits inside the device-timed region
    graph = torch.cuda.CUDAGraph()
    n0 = native.launch_count()
    with torch.cuda.graph(graph):
        backend.run_device(k, ptrs, torch.cuda.current_stream().cuda_stream)
    per_step = native.launch_count() - n0
    graph.replay()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        if flush is not None:
            flush.zero_()          # evict L2 between timed iterations (outside the events)
        starts[i].record(stream)
        graph.replay()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = per_step * steps
    # dominant kernel alone (the contraction launch, not its prepass / fold):
    # CUDA events placed by liblsb around that launch on the same stream
    kernel_ms = []
    native.profile(True)
    for _ in range(min(steps, 3)):
        if flush is not None:
            flush.zero_()
        backend.run_device(k, ptrs, sh)
        kernel_ms.append(native.last_kernel_ms())
    native.profile(False)
    times = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    res = {"ms_total": sum(times), "ms_mean": sum(times) / steps, "ms_min": min(times),
           "kernel_ms": sum(kernel_ms) / len(kernel_ms), "launches": launches,
           "steps": [s.kind + (f":{s.params['algo_selected']}" if s.params.get("algo_selected") else "")
                     for s in k.plan.steps],
           "kernel_launches_per_step": len(k.plan.steps)}

    if want_e2e:
        from paper_2205_00618_b200 import native as nt
        pinned = {}
        for s, a in host.items():
            pb = nt.PinnedBuffer(a.shape)
            pb.array[...] = a
            pinned[s] = pb
        bufs = {s: pb.array for s, pb in pinned.items()}
        outs = {s: nt.PinnedBuffer(k.slot_shapes[s]) for s in k.output_slots}
        for s, pb in outs.items():
            bufs[s] = pb.array
            if s in host:
                pb.array[...] = host[s]
        backend.execute(k, bufs)   # warm (allocates the kernel's device buffers)
        es, ee = [], []
        legacy = torch.cuda.default_stream()
        nsteps = max(1, min(steps, 5))
        for _ in range(nsteps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(legacy)
            backend.execute(k, bufs)
            b.record(legacy)
            torch.cuda.synchronize()
            es.append(a.elapsed_time(b))
        h2d = sum(host[s].nbytes for s in host)
        d2h = sum(int(np.prod(k.slot_shapes[s])) * 4 for s in k.output_slots)
        res["e2e_ms"] = sum(es) / len(es)
        res["h2d"], res["d2h"] = h2d, d2h
        for pb in list(pinned.values()) + list(outs.values()):
            pb.close()
    del tens
    return res


def traffic_of(name: str, steps) -> float | None:
    """dram read+write bytes per launch of the dominant kernel, from the
    committed `ncu --set full` capture of the same kernel/shape
    (profiles/traffic.json, written by tools/ncu_summary.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    algo = "tf32x3" if any("tf32x3" in s for s in steps) else "simt"
    ent = t.get(f"{name}_{algo}")
    return ent["dram_bytes_per_launch"] if ent else None


def roofline(steps, achieved, fp32_peak, sm_max, info, clocks, pk, name: str = "") -> dict:
    """Roofline of the dominant kernel (the contraction launch).

    3xTF32 path: three tf32 tcgen05 MMAs per fp32 product, so the ceiling for
    the algorithmic fp32 flops is TF32/3, TF32 = half the measured bf16 dense
    rate (MEASURED_PEAKS.json); the sustained figure because a step here is a
    long back-to-back run under the power cap.  SIMT path: FP32 FFMA peak."""
    fp32_note = (f"computed {info['sm_count']} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz "
                 "(MEASURED_PEAKS sm_max_mhz; no measured FP32 SIMT figure exists)")
    if any("tf32x3" in s for s in steps) and pk.get("bf16_tflops_sustained"):
        peak = pk["bf16_tflops_sustained"] / 2.0 / 3.0
        out = {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 2),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                "peak_source": "measured bf16 sustained (MEASURED_PEAKS) / 2 (tf32) / 3 (3xTF32 passes)",
                "peak_burst": round(pk.get("bf16_tflops", 0) / 6.0, 2),
                "fp32_simt_peak": round(fp32_peak, 2), "x_fp32_simt_peak": round(achieved / fp32_peak, 3),
                "kernel": "tf32x3_gemm_kernel (tcgen05.mma kind::tf32, TMEM, TMA)"}
        if achieved > peak:
            out["note"] = ("above the ceiling derived from the bf16 sustained figure: that rate was measured "
                           "under the power cap with bf16 MMAs; tf32 MMAs at the same clock draw less power, "
                           "so frac against peak_burst is the tighter bound here")
        return out
    return {"bound": "fp32", "achieved": round(achieved, 2), "peak": round(fp32_peak, 2),
            "unit": "TFLOP/s", "frac": round(achieved / fp32_peak, 4), "traffic": None,
            "peak_source": fp32_note,
            "frac_at_observed_clock": (round(achieved / (fp32_peak * clocks["sm_mhz"] / sm_max), 4)
                                       if clocks.get("sm_mhz") else None),
            "kernel": ("maxplus_cluster_kernel (FADD2+FMNMX3; 4-CTA cluster split-K, DSMEM max)"
                       if name == "C2" else "semiring_gemm_kernel (SIMT FFMA2 / FADD2+FMNMX3)")}


def time_gather(torch, world: int, rows: int, n: int, reps: int = 3) -> dict:
    """The optional NCCL all-gather of the C row shards: each
    rank's rows x n f32 shard into the full matrix on every rank through the
    library's lsb_allgather_rows (shard.gather_rows_native), timed on the
    device (CUDA events on the gather's stream, max over ranks).  Not part of
    `value`."""
    import torch.distributed as dist
    from paper_2205_00618_b200 import shard
    comm = shard.nccl_comm()
    local = torch.zeros((rows, n), dtype=torch.float32, device="cuda")
    out = torch.empty((rows * world, n), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    shard.gather_rows_native(comm, local, out, stream.cuda_stream)   # warm (NVLS setup)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        shard.gather_rows_native(comm, local, out, stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    recv = (world - 1) * rows * n * 4
    del local, out
    comm.close()
    return {"ms": round(ms, 4), "bytes_received_per_rank": recv,
            "algbw_GBps": round(recv / (ms * 1e-3) / 1e9, 1),
            "collective": "lsb_allgather_rows (ncclAllGather, library communicator)"}


def run_gpu(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ["LSB_DEVICE"] = str(local)
    torch.cuda.set_device(local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2205_00618_b200 import native
    native.init(local)
    info = native.device_info(local)
    pk = peaks()
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    fp32_peak = info["sm_count"] * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12   # TFLOP/s

    name = args.config
    with ClockSampler(local) as clk:
        res = gpu_config_run(name, args.steps, args.warmup, torch, rank, world,
                             flush_l2=(name != "C5"), want_e2e=True)
    clocks = clk.summary()
    flops_rank = FLOPS[name] // (world if name == "C5" else 1)
    total_flops = FLOPS[name] * (1 if name == "C5" else world)
    ms = res["ms_total"] / args.steps
    e2e_ms = res.get("e2e_ms", float("nan"))
    if world > 1:
        t = torch.tensor([ms, e2e_ms, res["ms_mean"]], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, e2e_ms, _ = t.tolist()
    value = total_flops / (ms * 1e-3) / 1e9
    gather = None
    if world > 1 and name == "C5":
        try:
            gather = time_gather(torch, world, CONFIGS[name]["M"] // world, CONFIGS[name]["M"])
            gather["value_with_gather"] = round(total_flops / ((ms + gather["ms"]) * 1e-3) / 1e9, 1)
        except Exception as e:  # report, never hide
            gather = {"error": f"{type(e).__name__}: {e}"}
    # roofline numerator: algorithmic flops of the dominant launch / its own
    # average duration (CUDA events around that launch, measured live)
    achieved = flops_rank / (res["kernel_ms"] * 1e-3) / 1e12

    per_config = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_per_config:
        for other in ("C1", "C2", "C3", "C4"):
            if other == name:
                continue
            try:
                r = gpu_config_run(other, max(args.steps, 10), args.warmup, torch, 0, 1,
                                   flush_l2=True, want_e2e=False)
                t = r["ms_mean"]
                g = FLOPS[other] / (t * 1e-3) / 1e9
                per_config[other] = {"desc": CONFIGS[other]["desc"], "GFLOP/s": round(g, 1),
                                     "ms": round(t, 4), "frac_fp32_peak": round(g / 1e3 / fp32_peak, 4),
                                     "kernels": r["steps"]}
                if CONFIGS[other].get("reduce") == "max":
                    # measured on this B200 (profiles/r01_ubench_pipes_maxplus.log):
                    # FADD2 and FMNMX3 share issue at 0.5 warp-instr/clk/SMSP, so
                    # one max-plus point (2 "flop") costs 1/32 of an SMSP cycle:
                    # the max-plus ceiling is half the FP32 FFMA peak
                    ceil = fp32_peak / 2.0
                    per_config[other]["maxplus_issue_ceiling_tflops"] = round(ceil, 2)
                    per_config[other]["frac_maxplus_ceiling"] = round(g / 1e3 / ceil, 4)
                if any("tf32x3" in s for s in r["steps"]) and pk.get("bf16_tflops_sustained"):
                    ceil = pk["bf16_tflops_sustained"] / 6.0
                    per_config[other]["frac_tf32x3_ceiling"] = round(g / 1e3 / ceil, 4)
                    if pk.get("bf16_tflops"):
                        # a sub-ms step runs at burst clocks: the tighter bound
                        per_config[other]["frac_tf32x3_burst_ceiling"] = round(g / 1e3 / (pk["bf16_tflops"] / 6.0), 4)
            except Exception as e:  # report, never hide
                per_config[other] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_time(name)
        except Exception as e:
            cpu = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": f"GFLOP/s, {name}: {CONFIGS[name]['desc']}",
            "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong" if name == "C5" else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic, seeded per SURVEY §8(d) (np.random.default_rng)",
            "config": {"workload": f"{name}: {CONFIGS[name]['desc']}",
                       "rows_per_rank": (CONFIGS[name].get("M", 0) // world) if name == "C5" else None,
                       "parallelism": f"row-shard x{world}" if world > 1 else "single",
                       "l2": "inputs 2 GiB > 126 MB L2" if name == "C5" else "L2 flushed between steps"},
            "roofline": {**roofline(res["steps"], achieved, fp32_peak, sm_max, info, clocks, pk, name),
                         "traffic": traffic_of(name, res["steps"]),
                         "kernel_ms": round(res["kernel_ms"], 4), "step_ms": round(res["ms_mean"], 4)},
            "e2e": {"value": round(total_flops / (e2e_ms * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                    "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": int(res.get("h2d", 0)), "d2h_bytes_per_step": int(res.get("d2h", 0)),
                    "path": "backend.execute (drop-in API) from pinned host buffers"},
            "gpu_launches": int(res["launches"]),
            "clocks": clocks,
        }
        if gather is not None:
            line["gather"] = gather
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if per_config:
            line["per_config"] = per_config
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_time(name, budget_s=args.ref_budget)
        if i >= args.warmup:
            vals.append(r)
    v = sum(x["value"] for x in vals) / len(vals)
    line = {"metric": f"GFLOP/s, {name}: {CONFIGS[name]['desc']}", "value": round(v, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "impl": "reference", "dtype": "f32",
            "data": "synthetic, seeded per SURVEY §8(d)",
            "config": {"workload": f"{name}: {CONFIGS[name]['desc']}"},
            "cpu_baseline": {**vals[-1], "value": round(v, 3)},
            "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": "reference CPU path = oracle/vmport.c, the C restatement of loopsmith's VM "
                    "arithmetic (bit-exact with it); the numba VM itself cannot travel to the box"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=6.0)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
