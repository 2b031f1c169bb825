#!/usr/bin/env python
"""Benchmark of the B200 loop-nest backend (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl b200|reference]

Metric: GFLOP/s per contraction config and fraction of the B200 roofline.
The headline line is the sharded config C5 (fp32 GEMM 16384^3, rows of A/C
split across the N ranks, B replicated, no data-path collective); at N=1 the
other configs C1..C4 are measured too and reported under "per_config".  A
"step" is one pass of the hot path over one batch of the synthetic input (one
full contraction).

Launch: ``--gpus N`` with N > 1 and no WORLD_SIZE in the environment re-runs
this script under ``torch.distributed.run`` (one rank per GPU, 127.0.0.1);
under an external torchrun WORLD_SIZE must equal --gpus.

value      device time (CUDA events on the launching stream, max over ranks),
           inputs resident in HBM; whole-job GFLOP/s = total flops / time.
e2e        the same contraction through the public drop-in API
           (backend.execute) from page-locked host buffers: H2D of the inputs,
           the kernels and D2H of the result inside the timed region.
           ``e2e.pageable`` repeats it from ordinary numpy arrays.
roofline   dominant kernel's achieved TFLOP/s (algorithmic 2*M*N*K / its own
           average launch duration, CUDA events placed by liblsb around that
           launch).  Tensor-core GEMM (fp16 hi/lo split of scaled operands):
           per 16-deep k block three K=16 fp16 MMAs (hi.hi, hi.lo, lo.hi), so
           the ceiling = measured bf16 dense BURST rate (MEASURED_PEAKS.json)
           / 3; also against the measured
           per-MHz bf16 rate (sustained run / its median clock) x the SM
           clock observed during the timed loop, and (for continuity with
           round 1) against the 3xTF32 ceiling bf16 / 6; SIMT path: the FP32
           peak 148 SMs x 128 lanes x 2 flop x sm_max_mhz.
clocks     NVML samples (SM clock, event reasons) taken only while the timed
           loop runs: median and minimum under load.
parity     each rank checks its own shard (sampled rows, f64 on the device)
           and, at N > 1, the all-gathered C; per-config runs check their full
           outputs (C1-C4) against f64.
cpu_baseline  oracle/vmport.c (C restatement of the reference VM arithmetic,
           bit-exact with it) on a bounded row sample, all host threads.
--impl reference   times that same CPU path as the reference arm, plus (when
           the reference package is installed under baseline/_ref) the real
           loopsmith VM on one core on the SURVEY §8(d) slice.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
#: C5 rows checked per shard against f64 (and per peer shard in the gathered C)
C5_CHECK_ROWS = 16


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- graphs / inputs

def load_graph(name: str, rows: int | None = None) -> dict:
    from paper_2205_00618_b200.shard import shard_graph
    with open(os.path.join(ROOT, "tests", "golden", "graphs", f"{GRAPH[name]}.json")) as f:
        obj = json.load(f)
    return shard_graph(obj, rows) if rows is not None else obj


def c5_rows(rows) -> np.ndarray:
    """Rows ``rows`` (sorted indices) of C5's A, drawn exactly as the full
    seeded matrix is (seed 4, 1024-row blocks in order)."""
    rng = np.random.default_rng(4)
    n, step = 16384, 1024
    out = np.empty((len(rows), n), np.float32)
    rows = np.asarray(rows)
    for lo in range(0, n, step):
        blk = rng.uniform(-1, 1, (step, n)).astype(np.float32)
        sel = (rows >= lo) & (rows < lo + step)
        out[sel] = blk[rows[sel] - lo]
        if lo + step > rows.max():
            break
    return out


def make_inputs(name: str, r0: int = 0, r1: int | None = None) -> dict:
    """Seeded inputs of SURVEY §8(d); for C5 only rows [r0, r1) of A."""
    if name == "C5":
        rng = np.random.default_rng(4)
        n = 16384
        r1 = n if r1 is None else r1
        # draw A row-block by row-block so a shard never holds all of A
        A = np.empty((r1 - r0, n), np.float32)
        step = 1024
        for lo in range(0, n, step):
            blk = rng.uniform(-1, 1, (step, n)).astype(np.float32)
            a, b = max(r0, lo), min(r1, lo + step)
            if a < b:
                A[a - r0:b - r0] = blk[a - lo:b - lo]
        B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        return {0: A, 1: B}
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import common
    if name == "C3":
        return common.config_inputs("C3g")
    return common.config_inputs(name)


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """NVML SM-clock / clock-event-reason samples on a background thread,
    started right before the timed loop and stopped right after it."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, torch, device: int, period_s: float = 0.005):
        self.period = period_s
        self.sm: list[float] = []
        self.reasons = 0
        self.max_mhz = None
        self.handle = None
        self.err = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            try:
                p = torch.cuda.get_device_properties(device)
                bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # report, never hide
            self.err = f"{type(e).__name__}: {e}"

    def _run(self):
        nv, h = self.nv, self.handle
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            except Exception as e:
                self.err = f"{type(e).__name__}: {e}"
                return
            time.sleep(self.period)

    def __enter__(self):
        self._stop = threading.Event()
        self._t = None
        if self.handle is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "error": self.err}
        return {"sm_mhz": statistics.median(self.sm), "sm_min_mhz": min(self.sm),
                "sm_max_mhz": self.max_mhz,
                "reasons": sorted(n for b, n in self.REASONS.items() if self.reasons & b),
                "samples": len(self.sm), "source": "NVML, timed loop only"}


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
            "cpu_model": cpu_model(),
            "sample": f"{name}: {sample} in {dt:.2f}s (oracle/vmport.c, VM f32 arithmetic)"}


#: SURVEY §8(d) slices the reference VM is timed on (rows of the output)
VM_SLICE = {"C1": None, "C2": None, "C3": 1, "C4": 128, "C5": 8}


def reference_vm_time(name: str, min_ms: float = 500.0) -> dict:
    """The real loopsmith VM (numba, single-threaded: 1 core) through its own
    public API -- ``feedback.benchmark(compile_tree(lower(g)), buffers)``
    (feedback.py:270-295) -- on the SURVEY §8(d) slice of ``name`` with the
    §8(d) schedule (the graphs' own), extrapolated linearly to the full
    config.  Needs the reference installed under baseline/_ref."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "loopsmith")):
        return {"unavailable": "baseline/_ref has no loopsmith install (tools/run_refsuite.sh install)"}
    os.environ.setdefault("NUMBA_NUM_THREADS", "1")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import loopsmith as ls
    from loopsmith import feedback, serialize, vm
    from paper_2205_00618_b200.shard import shard_graph
    t0 = time.perf_counter()
    vm.warmup()
    warm_s = time.perf_counter() - t0
    # C3: the host-padded valid-conv form SURVEY §8(d) times (X [8,64,58,58])
    with open(os.path.join(ROOT, "tests", "golden", "graphs", f"{name}.json")) as f:
        gobj = json.load(f)
    frac = 1.0
    if name == "C3":
        # one image of eight: the batch var n resized to 1
        gobj = shard_graph(gobj, 1, var_name="n")
        frac = 1 / 8
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import common
        full = common.config_inputs("C3")
        bufs = {0: full[0][:1].copy(), 1: full[1]}
    elif VM_SLICE[name]:
        rows = VM_SLICE[name]
        gobj = shard_graph(gobj, rows, var_name="b" if name == "C4" else "m")
        frac = rows / CONFIGS[name]["M"]
        full = make_inputs(name, 0, rows) if name == "C5" else make_inputs(name)
        bufs = {s: (a[:rows].copy() if s == 0 else a) for s, a in full.items()}
    else:
        bufs = make_inputs(name)
    g = serialize.loads(json.dumps(gobj))
    kern = ls.compile_tree(ls.lower(g), ls.avx512_like() if name != "C3" else ls.avx2_like())
    res = feedback.benchmark(kern, bufs, min_ms=min_ms)
    ms = float(res.elapsed_ms) / max(int(res.repeats), 1)
    flops = FLOPS[name] * frac
    return {"value": round(flops / (ms * 1e-3) / 1e9, 4), "unit": "GFLOP/s", "cores": 1,
            "kind": "reference", "cpu_model": cpu_model(),
            "sample": (f"{name}: loopsmith VM (numba, 1 thread) via feedback.benchmark, "
                       f"{frac:.6g} of the config ({ms:.2f} ms per call), extrapolated linearly"),
            "numba_warmup_s": round(warm_s, 1)}


# ---------------------------------------------------------------- GPU arm

def _check_rows(torch, A_rows, B, got_rows, rule: str) -> dict:
    """f64 on the device: ``got_rows`` vs A_rows @ B (or max-plus)."""
    a, b = A_rows.double(), B.double()
    if rule == "maxplus":
        ref = torch.stack([(a[i][:, None] + b).amax(0) for i in range(a.shape[0])])
        same = torch.equal(got_rows, ref.float())
        return {"bitexact": bool(same), "rows": int(a.shape[0])}
    ref = a @ b
    return _tol(torch, got_rows.double(), ref)


def _tol(torch, got, ref) -> dict:
    d = (got - ref).abs()
    # the reference's acceptance formula, per element (test_acceptance.py:57-58);
    # max_err_rel_max_ref is the laxer max|d| / max(max|ref|, 1)
    metric = float((d / ref.abs().clamp(min=1.0)).max())
    lax = float(d.max() / torch.clamp(ref.abs().max(), min=1.0))
    strict = float((d <= 1e-5 + 1e-4 * ref.abs()).double().mean())
    return {"ref_metric": metric, "max_err_rel_max_ref": lax, "strict_pass": strict, "ok": metric <= 1e-4,
            "elements": int(ref.numel())}


def config_parity(torch, name: str, tens: dict) -> dict:
    """Full-output check of a per-config run against f64 on the device:
    C2 bit-exact vs float32(f64), C1/C3/C4 the strict per-element rule and
    the reference metric."""
    if name == "C2":
        A, B, C = tens[0], tens[1], tens[2]
        ok = True
        for r in range(0, A.shape[0], 64):
            ref = (A[r:r + 64].double()[:, :, None] + B.double()[None]).amax(1).float()
            ok &= torch.equal(C[r:r + 64], ref)
        return {"rule": "bit-exact vs float32(f64)", "bitexact": bool(ok), "elements": int(C.numel())}
    if name == "C3":
        import torch.nn.functional as F
        x, w, o = tens[0].double(), tens[1].double(), tens[2].double()
        ref = F.conv2d(x, w, padding=1)
        return {"rule": "|d|<=1e-5+1e-4|ref|", **_tol(torch, o.reshape(ref.shape), ref)}
    A, B = tens[0].double(), tens[1].double()
    ref = A @ B
    if name == "C4":
        ref = torch.relu(ref + tens[2].double()[None, :])
        C = tens[3]
    else:
        C = tens[2]
    return {"rule": "|d|<=1e-5+1e-4|ref|", **_tol(torch, C.double().reshape(ref.shape), ref)}


def gpu_config_run(name: str, steps: int, warmup: int, torch, rank: int, world: int,
                   flush_l2: bool, want_e2e: bool):
    from paper_2205_00618_b200 import backend, native, shard
    cfg = CONFIGS[name]
    if name == "C5":
        r0, r1 = shard.shard_rows(cfg["M"], world, rank)
        graph = load_graph("C5", rows=r1 - r0)
        host = make_inputs("C5", r0, r1)
    else:
        r0, r1 = 0, cfg.get("M", 0)
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
    cgraph = torch.cuda.CUDAGraph()
    n0 = native.launch_count()
    with torch.cuda.graph(cgraph):
        backend.run_device(k, ptrs, torch.cuda.current_stream().cuda_stream)
    per_step = native.launch_count() - n0
    cgraph.replay()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch, torch.cuda.current_device()) as clk:
        for i in range(steps):
            if flush is not None:
                flush.zero_()          # evict L2 between timed iterations (outside the events)
            starts[i].record(stream)
            cgraph.replay()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = per_step * steps
    times = [s.elapsed_time(e) for s, e in zip(starts, ends)]
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
    torch.cuda.synchronize()
    res = {"ms_total": sum(times), "ms_mean": sum(times) / steps, "ms_min": min(times),
           "kernel_ms": sum(kernel_ms) / len(kernel_ms), "launches": launches,
           "clocks": clk.summary(),
           "steps": [s.kind + (f":{s.params['algo_selected']}" if s.params.get("algo_selected") else "")
                     for s in k.plan.steps],
           "kernel_launches_per_step": len(k.plan.steps)}

    # parity of what the timed steps computed (outputs are deterministic)
    if name == "C5":
        rows = r1 - r0
        idx = sorted(set(np.linspace(0, rows - 1, C5_CHECK_ROWS).astype(int).tolist()))
        sel = torch.tensor(idx, device=dev)
        res["parity"] = {"rank": rank, "rows": [r0, r1], "checked_rows": len(idx),
                         **_check_rows(torch, tens[0][sel], tens[1], tens[2][sel], "sum")}
        res["C"] = tens[2]
        res["B"] = tens[1]
    else:
        res["parity"] = config_parity(torch, name, tens)

    if want_e2e:
        res["e2e"] = e2e_run(k, host, steps, torch)
    if name != "C5":
        del tens
    return res


def e2e_run(k, host: dict, steps: int, torch) -> dict:
    """The same contraction through ``backend.execute`` (the drop-in call)
    with host buffers: ordinary numpy arrays (pageable) and page-locked
    ones.  Each timed call includes H2D of the inputs and D2H of the output
    (CUDA events on the legacy stream around the call, host-synchronised)."""
    from paper_2205_00618_b200 import backend
    from paper_2205_00618_b200 import native as nt
    legacy = torch.cuda.default_stream()
    nsteps = max(1, min(steps, 5))

    def timed(bufs):
        backend.execute(k, bufs)   # warm: device buffers, host registration
        es = []
        for _ in range(nsteps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(legacy)
            backend.execute(k, bufs)
            b.record(legacy)
            torch.cuda.synchronize()
            es.append(a.elapsed_time(b))
        return sum(es) / len(es)

    out = {}
    if torch.distributed.is_available() and torch.distributed.is_initialized() and \
            torch.distributed.get_world_size() > 1:
        # N > 1: the contract's pinned figure only (every rank staging 3 GiB
        # through its own 512 MiB pinned ring at once would measure host RAM)
        out["pageable_ms"] = float("nan")
        out["pageable_first_call_ms"] = float("nan")
        pageable = False
    else:
        pageable = True
    # pageable: the caller's own numpy arrays (fresh output arrays)
    bufs = {s: a for s, a in host.items()} if pageable else {}
    if pageable:
        for s in k.output_slots:
            bufs[s] = np.empty(k.slot_shapes[s], np.float32) if s not in host else host[s].copy()
        t0 = time.perf_counter()
        backend.execute(k, dict(bufs))
        first = (time.perf_counter() - t0) * 1e3
        out["pageable_ms"] = timed(bufs)
        out["pageable_first_call_ms"] = first
    del bufs
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
    out["pinned_ms"] = timed(bufs)
    for pb in list(pinned.values()) + list(outs.values()):
        pb.close()
    out["h2d"] = sum(host[s].nbytes for s in host)
    out["d2h"] = sum(int(np.prod(k.slot_shapes[s])) * 4 for s in k.output_slots)
    return out


def gathered_parity(torch, world: int, rank: int, C_local, B, comm_out) -> dict:
    """Check the all-gathered C: this rank's rows equal its local shard
    bit-for-bit, and sampled rows of the next rank's shard match f64."""
    from paper_2205_00618_b200 import shard
    M = comm_out.shape[0]
    r0, r1 = shard.shard_rows(M, world, rank)
    own = bool(torch.equal(comm_out[r0:r1], C_local))
    peer = (rank + 1) % world
    p0, p1 = shard.shard_rows(M, world, peer)
    idx = sorted(set(np.linspace(p0, p1 - 1, 4).astype(int).tolist()))
    A = torch.from_numpy(c5_rows(idx)).to(C_local.device)
    chk = _check_rows(torch, A, B, comm_out[torch.tensor(idx, device=C_local.device)], "sum")
    return {"own_rows_bitexact": own, "peer": peer, "peer_rows_checked": len(idx), **chk}


def traffic_of(name: str, steps) -> float | None:
    """dram read+write bytes per launch of the dominant kernel, from the
    committed `ncu --set full` capture of the same kernel/shape
    (profiles/traffic.json, written by tools/ncu_summary.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    algo = "tf32x3" if any("tf32x3" in s for s in steps) else "conv" if any(s.startswith("conv") for s in steps) \
        else "simt"
    ent = t.get(f"{name}_{algo}")
    return ent["dram_bytes_per_launch"] if ent else None


def _frac_clock(achieved, pk, obs, div):
    """achieved / the measured bf16 dense rate per MHz (MEASURED_PEAKS: the
    sustained run and its median SM clock under load) x the SM clock seen
    during this timed loop, / div (3 = three fp16 MMAs per fp32 MAC)."""
    rate = pk.get("bf16_tflops_sustained")
    clk = (pk.get("clocks_under_load") or {}).get("sm_mhz_median")
    if not (rate and clk and obs):
        return None
    return round(achieved / (rate / clk * obs / div), 4)


def roofline(steps, achieved, fp32_peak, sm_max, info, clocks, pk, name: str = "") -> dict:
    """Roofline of the dominant kernel (the contraction launch).

    Tensor-core GEMM: the fp16 hi/lo split runs three kind::f16 MMAs (hi.hi,
    hi.lo, lo.hi) per fp32 product, so the ceiling for the algorithmic fp32
    flops is the measured bf16 dense BURST rate / 3 (MEASURED_PEAKS.json,
    taken near sm_max_mhz); ``frac`` is against it,
    ``frac_at_observed_clock`` against the measured per-MHz rate at the median
    SM clock seen during the timed loop, ``frac_3xtf32_ceiling`` against the
    round-1 algorithm's bf16 / 6.  SIMT path: FP32 peak."""
    fp32_note = (f"computed {info['sm_count']} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz "
                 "(MEASURED_PEAKS sm_max_mhz; no measured FP32 SIMT figure exists)")
    obs = clocks.get("sm_mhz")
    if any("tf32x3" in s for s in steps) and pk.get("bf16_tflops"):
        peak = pk["bf16_tflops"] / 3.0
        out = {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 2),
               "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
               "peak_source": ("measured bf16 dense burst (MEASURED_PEAKS bf16_tflops) / 3: three fp16 "
                               "K=16 MMAs (hi.hi, hi.lo, lo.hi) per fp32 product"),
               "frac_at_observed_clock": _frac_clock(achieved, pk, obs, 3.0),
               "peak_sustained": round(pk.get("bf16_tflops_sustained", 0) / 3.0, 2),
               "frac_3xtf32_ceiling": round(achieved / (pk["bf16_tflops"] / 6.0), 4),
               "fp32_simt_peak": round(fp32_peak, 2), "x_fp32_simt_peak": round(achieved / fp32_peak, 3),
               "kernel": "tf32x3_gemm_kernel (tcgen05.mma kind::f16 x3 split, TMEM, TMA)"}
        return out
    return {"bound": "fp32", "achieved": round(achieved, 2), "peak": round(fp32_peak, 2),
            "unit": "TFLOP/s", "frac": round(achieved / fp32_peak, 4), "traffic": None,
            "peak_source": fp32_note,
            "frac_at_observed_clock": (round(achieved / (fp32_peak * obs / sm_max), 4) if obs else None),
            "kernel": ("maxplus kernel (FADD2+FMNMX3)" if name == "C2"
                       else "semiring_gemm_kernel (SIMT FFMA2 / FADD2+FMNMX3)")}


def time_gather(torch, world: int, rows: int, n: int, reps: int = 3, local=None) -> dict:
    """The optional NCCL all-gather of the C row shards: each
    rank's rows x n f32 shard into the full matrix on every rank through the
    library's lsb_allgather_rows (shard.gather_rows_native), timed on the
    device (CUDA events on the gather's stream, max over ranks).  Not part of
    `value`.  With ``local`` (the computed shard) the gathered matrix is
    returned for checking."""
    import torch.distributed as dist
    from paper_2205_00618_b200 import shard
    comm = shard.nccl_comm()
    if local is None:
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
    comm.close()
    return {"ms": round(ms, 4), "bytes_received_per_rank": recv,
            "algbw_GBps": round(recv / (ms * 1e-3) / 1e9, 1),
            "collective": "lsb_allgather_rows (ncclAllGather, library communicator)",
            "_out": out}


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
    res = gpu_config_run(name, args.steps, args.warmup, torch, rank, world,
                         flush_l2=(name != "C5"), want_e2e=True)
    clocks = res["clocks"]
    sharded = name == "C5"
    flops_rank = FLOPS[name] // (world if sharded else 1)
    total_flops = FLOPS[name] * (1 if sharded else world)
    ms = res["ms_total"] / args.steps
    e2e = res["e2e"]
    e2e_ms, e2e_pin_ms = e2e["pageable_ms"], e2e["pinned_ms"]
    parity = res["parity"]
    if world > 1:
        t = torch.tensor([ms, e2e_ms, e2e_pin_ms, res["kernel_ms"]], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, e2e_ms, e2e_pin_ms, _ = t.tolist()
        box = [None] * world
        torch.distributed.all_gather_object(box, {"parity": parity, "clocks": clocks})
        parity = {"per_rank": [b["parity"] for b in box],
                  "ok": all(b["parity"].get("ok", False) for b in box)}
        clocks = {**clocks, "per_rank_sm_mhz": [b["clocks"].get("sm_mhz") for b in box],
                  "reasons": sorted({r for b in box for r in b["clocks"].get("reasons", [])})}
    value = total_flops / (ms * 1e-3) / 1e9
    gather = None
    if world > 1 and sharded:
        try:
            rows = res["C"].shape[0]
            gather = time_gather(torch, world, rows, CONFIGS[name]["N"], local=res["C"])
            out = gather.pop("_out")
            gp = gathered_parity(torch, world, rank, res["C"], res["B"], out)
            del out
            box = [None] * world
            torch.distributed.all_gather_object(box, gp)
            gather["parity"] = {"per_rank": box,
                                "ok": all(b["own_rows_bitexact"] and b["ok"] for b in box)}
            gather["value_with_gather"] = round(total_flops / ((ms + gather["ms"]) * 1e-3) / 1e9, 1)
        except Exception as e:  # report, never hide
            gather = {"error": f"{type(e).__name__}: {e}"}
    res.pop("C", None)
    res.pop("B", None)
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
                kt = FLOPS[other] / (r["kernel_ms"] * 1e-3) / 1e12
                per_config[other] = {"desc": CONFIGS[other]["desc"], "GFLOP/s": round(g, 1),
                                     "ms": round(t, 4), "kernel_ms": round(r["kernel_ms"], 4),
                                     "frac_fp32_peak": round(g / 1e3 / fp32_peak, 4),
                                     "kernels": r["steps"], "parity": r["parity"],
                                     "clocks_sm_mhz": r["clocks"].get("sm_mhz")}
                if CONFIGS[other].get("reduce") == "max":
                    # measured on this B200 (profiles/r01_ubench_pipes_maxplus.log):
                    # FADD2 and FMNMX3 share issue at 0.5 warp-instr/clk/SMSP, so
                    # one max-plus point (2 "flop") costs 1/32 of an SMSP cycle:
                    # the max-plus ceiling is half the FP32 FFMA peak
                    ceil = fp32_peak / 2.0
                    per_config[other]["maxplus_issue_ceiling_tflops"] = round(ceil, 2)
                    per_config[other]["frac_maxplus_ceiling"] = round(g / 1e3 / ceil, 4)
                    per_config[other]["kernel_frac_maxplus_ceiling"] = round(kt / ceil, 4)
                if pk.get("bf16_tflops") and (any("tf32x3" in s for s in r["steps"]) or other == "C3"):
                    # the GEMM's algorithm ceiling is bf16 / 3 (see roofline());
                    # the conv keeps the 3xTF32 ceiling bf16 / 6 as its yardstick
                    # (its MMA mix: two tf32 + one fp16-class MMA per 16 channels
                    # of 64 filters on 128 rows, rows half wasted by the stacking)
                    ceil = pk["bf16_tflops"] / (6.0 if other == "C3" else 3.0)
                    per_config[other]["tensor_ceiling_tflops"] = round(ceil, 2)
                    per_config[other]["frac_tensor_ceiling"] = round(g / 1e3 / ceil, 4)
                    per_config[other]["kernel_frac_tensor_ceiling"] = round(kt / ceil, 4)
                    per_config[other]["frac_3xtf32_ceiling"] = round(g / 1e3 / (pk["bf16_tflops"] / 6.0), 4)
                tr = traffic_of(other, r["steps"])
                if tr is not None:
                    per_config[other]["traffic"] = tr
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
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic, seeded per SURVEY §8(d) (np.random.default_rng)",
            "config": {"workload": f"{name}: {CONFIGS[name]['desc']}",
                       "rows_per_rank": (CONFIGS[name]["M"] // world) if sharded else None,
                       "parallelism": f"row-shard x{world}" if world > 1 else "single",
                       "l2": "inputs 2 GiB > 126 MB L2" if name == "C5" else "L2 flushed between steps"},
            "roofline": {**roofline(res["steps"], achieved, fp32_peak, sm_max, info, clocks, pk, name),
                         "traffic": traffic_of(name, res["steps"]),
                         "kernel_ms": round(res["kernel_ms"], 4), "step_ms": round(res["ms_mean"], 4)},
            "e2e": {"value": round(total_flops / (e2e_pin_ms * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                    "ms_per_step": round(e2e_pin_ms, 3),
                    "h2d_bytes_per_step": int(e2e["h2d"]), "d2h_bytes_per_step": int(e2e["d2h"]),
                    "path": "backend.execute (drop-in API) from page-locked host buffers",
                    "pageable": ({"value": round(total_flops / (e2e_ms * 1e-3) / 1e9, 1),
                                  "ms_per_step": round(e2e_ms, 3),
                                  "first_call_ms": round(e2e["pageable_first_call_ms"], 1),
                                  "path": "backend.execute from ordinary numpy arrays (pageable)"}
                                 if world == 1 else None)},
            "gpu_launches": int(res["launches"]),
            "clocks": clocks,
            "parity": parity,
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
                    "arithmetic (bit-exact with it) on all host threads; reference_vm = the "
                    "loopsmith VM itself (numba, 1 thread) on the SURVEY §8(d) slice"}
    if not args.no_vm:
        try:
            line["reference_vm"] = reference_vm_time(name)
        except Exception as e:  # report, never hide
            line["reference_vm"] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(nproc: int, argv: list[str]) -> int:
    """Re-run this script as ``nproc`` ranks under torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1); returns the launcher's exit
    code.  Rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + argv
    env = {**os.environ, "LSB_BENCH_LAUNCHED": "1"}
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-vm", action="store_true", help="reference arm: skip the loopsmith VM timing")
    ap.add_argument("--launch", action="store_true",
                    help="go through the torch.distributed.run launcher even for --gpus 1")
    ap.add_argument("--ref-budget", type=float, default=6.0)
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1 or args.launch:
            sys.exit(launch_ranks(args.gpus, [a for a in argv if a != "--launch"]))
    elif int(os.environ["WORLD_SIZE"]) != args.gpus:
        log(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}")
        sys.exit(2)
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
