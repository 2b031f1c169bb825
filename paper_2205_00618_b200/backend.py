"""Drop-in B200 replacement for ``loopsmith.backend`` (compile-then-call).

Public surface, same names / arguments / errors as the reference
(reference pkg/src/loopsmith/backend.py):

  compile_tree(tree, target, unroll_limit=None, interleave=True)  backend.py:1427-1454
  compile(...)                      alias                          backend.py:1496-1500
  compile_single_operand(tree, target, unroll_limit=None)          backend.py:1503-1514
  execute(kernel, buffers)                                         backend.py:121-161
  CompiledKernel                                                   backend.py:92-118
  BlockTooLarge / HasReduction / ShapeMismatch                     backend.py:41-46, feedback.py:21

Differences by design: ``program`` is a launch program (one record per
sm_100a kernel launch) instead of a VM instruction list; ``target`` (a CPU
vector-ISA preset) is accepted and ignored -- tiles come from the B200 kernel
set, with split factors used only as hints.  ``execute`` copies host buffers
to HBM, launches, and copies outputs back; ``run_device`` runs on
caller-owned device buffers (inputs already resident).

There is no CPU path: without liblsb.so or a CUDA device every call raises.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import native, render
from .errors import BlockTooLarge, HasReduction, ShapeMismatch
from .graph import Graph
from .planner import Plan, Ref, Step, plan_graph
from .schedule import alloc_scratch_bytes, schedule_counters

#: reference program.py:186-190 counter names (kept so callers that read
#: kernel.counters / memory_access_count() keep working)
COUNTERS = ("vload", "vload.strided", "vbroadcast", "vstore", "sload",
            "sstore", "vop", "vfma", "vreduce", "sop", "sfma", "post",
            "vbroadcast.imm", "loop")
MEM_COUNTERS = ("vload", "vload.strided", "vbroadcast", "vstore", "sload", "sstore")

__all__ = ["compile_tree", "compile", "compile_single_operand", "compile_graph", "execute",
           "run_device", "CompiledKernel", "BlockTooLarge", "HasReduction", "ShapeMismatch"]


# ---------------------------------------------------------------------------
# the compiled artifact
# ---------------------------------------------------------------------------

@dataclass
class LaunchRecord:
    op: str            # "launch.gemm" | "launch.conv" | "launch.nest"
    step: Step


@dataclass(frozen=True)
class RegionInfo:
    """program.py:81-91 RegionInfo for a contraction launch (instruction
    index = launch index): ``accum_regs`` are the schedule's register block
    counted in the target's vector registers, as the reference counts its
    accumulators (backend.py:593-691).  The device kernel keeps its
    accumulators in registers (SIMT) or TMEM (tcgen05) for the whole
    reduction: no spills, one store per output at the epilogue."""
    node: int
    start: int
    end: int
    accum_regs: tuple
    prologue_end: int
    epilogue_start: int


@dataclass
class LaunchProgram:
    """Stands in for program.KernelProgram: one record per kernel launch."""
    instrs: list[LaunchRecord]
    lanes: int = 32
    vregs: int = 255
    regions: list = field(default_factory=list)
    buffers: list = field(default_factory=list)
    var_names: list = field(default_factory=list)

    def disassemble(self) -> str:
        """One block per launch: the header, then the loop nest the kernel
        executes (render.py).  ``algo`` is known once descriptors are built
        (first execute / run_device)."""
        out = []
        for r in self.instrs:
            algo = r.step.params.get("algo_selected")
            out.append(render.render_step(r.step, f"{r.op} {r.step.describe()}" + (f" algo={algo}" if algo else "")))
        return "".join(out)

    def encode(self):
        raise NotImplementedError("B200 launch programs are not VM-encodable")


@dataclass
class CompiledKernel:
    """Same fields callers read on the reference's CompiledKernel
    (backend.py:92-118, cli.py:56-72, session.py:247-250, tuner.py:66-69)."""
    program: LaunchProgram
    target: object
    slot_shapes: dict[int, tuple[int, ...]]
    input_slots: set[int]
    output_slots: set[int]
    scratch_bytes: int
    compile_ms: float
    flops: int
    dfg_bytes_moved: int
    unrolled_spans: list = field(default_factory=list)
    unroll_limit: int = 0
    counters: dict[str, int] = field(default_factory=dict)
    plan: Optional[Plan] = None
    _runner: object = None

    def disassemble(self) -> str:
        return self.program.disassemble()

    def memory_access_count(self) -> int:
        return sum(self.counters.get(k, 0) for k in MEM_COUNTERS)

    def _count(self, launches: int) -> None:
        """Counters of the last execution (reset per call, like the VM's
        backend.py:121-161): kernel launches, one ``loop`` per launch; for
        contractions the schedule's memory instructions as register-blocked
        16-byte vector code (schedule.schedule_counters: vload / vbroadcast /
        vstore depend on the splits and the loop order, so the tuner can rank
        schedules), for other launches the modeled 16-byte global traffic
        (render.traffic)."""
        c = {k: 0 for k in COUNTERS}
        for st in self.plan.steps:
            sm = st.params.get("schedule")
            if st.kind == "gemm" and sm is not None:
                p = st.params
                ld, bc, stv = schedule_counters(sm, p["M"], p["N"], p["K"], p["batch"])
                c["vload"] += ld
                c["vbroadcast"] += bc
                c["vstore"] += stv
            else:
                ld, stv = render.traffic(st)
                c["vload"] += ld
                c["vstore"] += stv
            c["loop"] += 1
        c["launches"] = launches
        self.counters = c

    @property
    def runner(self) -> "Runner":
        if self._runner is None:
            self._runner = Runner(self.plan)
        return self._runner


# ---------------------------------------------------------------------------
# compile
# ---------------------------------------------------------------------------

def _compile(graph: Graph, target, unroll_limit, tree=None) -> CompiledKernel:
    t0 = time.perf_counter()
    plan = plan_graph(graph)
    prog = LaunchProgram([LaunchRecord(f"launch.{s.kind}", s) for s in plan.steps],
                         lanes=getattr(target, "lanes", 32), vregs=getattr(target, "vregs", 255))
    for st in plan.steps:
        if st.kind == "gemm":
            _resolve_algo(st)
    lanes, vregs = getattr(target, "lanes", 16), getattr(target, "vregs", 32)
    for i, st in enumerate(plan.steps):
        sm = st.params.get("schedule")
        if sm is not None:
            block = min(sm.block, max(1, (vregs - 8) * lanes))
            prog.regions.append(RegionInfo(sm.node, i, i + 1, tuple(range(-(-block // lanes))), i, i))
    ms = (time.perf_counter() - t0) * 1000.0
    limit = unroll_limit if unroll_limit is not None else getattr(target, "unroll_limit", 0)
    # scratch: the schedule's materialized allocations by the reference's rule
    # (staged operand panels, unfused intermediates) when compiled from a
    # lowered tree, at least the device scratch this plan allocates
    scratch = max(plan.scratch_bytes, alloc_scratch_bytes(tree) or 0)
    return CompiledKernel(program=prog, target=target, slot_shapes=plan.slot_shapes,
                          input_slots=set(plan.input_slots), output_slots=set(plan.output_slots),
                          scratch_bytes=scratch, compile_ms=ms,
                          flops=graph.count_flops(), dfg_bytes_moved=graph.bytes_moved(),
                          unroll_limit=limit, counters={k: 0 for k in COUNTERS}, plan=plan)


def _resolve_algo(step: Step) -> None:
    """The algorithm lsb_semiring_gemm will pick (lsb_gemm_algo, host-only
    heuristics), recorded for disassembly; left unset without the library."""
    p = step.params
    d = native.GemmDesc()
    d.M, d.N, d.K, d.batch = p["M"], p["N"], p["K"], p["batch"]
    d.combine, d.reduce, d.beta_in_loop = p["combine"], p["reduce"], p["beta_in_loop"]
    d.algo = p.get("algo", 0)
    d.tile_m, d.tile_n, d.split_k = p.get("tile_m", 0), p.get("tile_n", 0), p.get("split_k", 0)
    d.m_begin, d.m_end = p.get("m_begin", 0), p.get("m_end", 0)
    try:
        p["algo_selected"] = native.gemm_algo(d)
    except (OSError, native.NativeError):
        pass


def compile_tree(tree, target=None, unroll_limit: Optional[int] = None,
                 interleave: bool = True) -> CompiledKernel:
    """Compile a lowered loop tree (reference LoopTree) for the B200.

    Only ``tree.dfg`` is consumed: every schedule annotation is
    value-preserving (feedback.py:69-75), so split factors are tile hints."""
    del interleave
    return _compile(Graph.coerce(tree), target, unroll_limit,
                    tree if hasattr(tree, "alloc") else None)


def compile(tree, target=None, unroll_limit: Optional[int] = None,  # noqa: A001
            interleave: bool = True) -> CompiledKernel:
    """Alias of ``compile_tree`` (backend.py:1496-1500)."""
    return compile_tree(tree, target, unroll_limit, interleave)


def compile_single_operand(tree, target=None, unroll_limit: Optional[int] = None) -> CompiledKernel:
    """Reduction-free single-input trees (backend.py:1503-1514)."""
    g = Graph.coerce(tree)
    for n in g.nodes.values():
        red = g.reduction_dims(n)
        if red:
            raise HasReduction(f"node {n.id} reduces {[g.vars[v].name for v in red]}")
    n_reads = sum(1 for n in g.nodes.values() if n.kind == "read")
    if n_reads != 1:
        raise ValueError(f"single-operand tree must have 1 input, has {n_reads}")
    return _compile(g, target, unroll_limit, tree if hasattr(tree, "alloc") else None)


def compile_graph(graph, target=None) -> CompiledKernel:
    """Compile from a DFG, the reference's canonical graph JSON (dict / str,
    serialize.py:32-87) or a Graph mirror -- the path the CLI data format
    and the GPU-box parity fixtures use."""
    return _compile(Graph.coerce(graph), target, None)


# ---------------------------------------------------------------------------
# runtime: device buffers + descriptors
# ---------------------------------------------------------------------------

def _current_device() -> int:
    return int(os.environ.get("LSB_DEVICE", os.environ.get("LOCAL_RANK", "0")))


class Runner:
    """Launches a plan.  Owns scratch buffers (and, for ``execute``, device
    copies of the external slots); descriptors are rebuilt only when the
    buffer pointers change."""

    def __init__(self, plan: Plan, device: Optional[int] = None):
        self.plan = plan
        self.device = _current_device() if device is None else device
        native.init(self.device)
        self.scratch = {k: native.DeviceBuffer(4 * n) for k, n in plan.scratch.items()}
        self.slot_bufs: dict[int, native.DeviceBuffer] = {}
        self._descs = None
        self._desc_key = None

    def slot_buffers(self) -> dict[int, int]:
        for slot, shape in self.plan.slot_shapes.items():
            if slot not in self.slot_bufs:
                n = int(np.prod(shape)) if shape else 1
                self.slot_bufs[slot] = native.DeviceBuffer(4 * n)
        return {s: b.ptr for s, b in self.slot_bufs.items()}

    def _ptr(self, slots: dict[int, int], ref_base) -> int:
        ref, base = ref_base
        if ref.kind == "slot":
            p = slots[ref.key]
        else:
            p = self.scratch[ref.key].ptr
        return int(p) + 4 * int(base)

    def _acc_ptr(self, slots, acc) -> int:
        return self._ptr(slots, (acc.ref, acc.base))

    def _epi(self, slots, step: Step, arr) -> int:
        for i, e in enumerate(step.epi):
            st = arr[i]
            st.combine, st.reduce, st.pre, st.post = e.combine, e.reduce, e.pre, e.post
            st.beta, st.alpha = e.beta, e.alpha
            strides = step.params["epi_strides"][i]
            if e.operand is not None:
                st.operand = self._acc_ptr(slots, e.operand)
                for d, v in enumerate(strides["operand"]):
                    st.so[d] = v
            if e.c_in is not None:
                st.c_in = self._acc_ptr(slots, e.c_in)
                for d, v in enumerate(strides["c_in"]):
                    st.sc[d] = v
        return len(step.epi)

    def _build(self, slots: dict[int, int]):
        descs = []
        for step in self.plan.steps:
            p = step.params
            if step.kind == "gemm":
                d = native.GemmDesc()
                d.M, d.N, d.K, d.batch = p["M"], p["N"], p["K"], p["batch"]
                d.A = self._ptr(slots, p["A"]); d.sa_b, d.sa_m, d.sa_k = p["sa_b"], p["sa_m"], p["sa_k"]
                d.B = self._ptr(slots, p["B"]); d.sb_b, d.sb_k, d.sb_n = p["sb_b"], p["sb_k"], p["sb_n"]
                d.C = self._ptr(slots, p["C"]); d.sc_b, d.sc_m, d.sc_n = p["sc_b"], p["sc_m"], p["sc_n"]
                d.combine, d.reduce = p["combine"], p["reduce"]
                d.beta, d.beta_in_loop = p["beta"], p["beta_in_loop"]
                d.n_epi = self._epi(slots, step, d.epi)
                d.algo = p.get("algo", 0)
                d.split_k = p.get("split_k", 0)
                d.tile_m, d.tile_n = p.get("tile_m", 0), p.get("tile_n", 0)
                d.m_begin, d.m_end = p.get("m_begin", 0), p.get("m_end", 0)
                p["algo_selected"] = native.gemm_algo(d)
                descs.append((native.semiring_gemm, d))
            elif step.kind == "conv":
                d = native.ConvDesc()
                for k in ("N", "C", "H", "W", "CO", "R", "S", "HO", "WO", "stride_h", "stride_w",
                          "pad_h", "pad_w", "dil_h", "dil_w"):
                    setattr(d, k, p[k])
                d.fill = p["fill"]
                d.x = self._ptr(slots, p["x"]); d.w = self._ptr(slots, p["w"]); d.o = self._ptr(slots, p["o"])
                for i in range(4):
                    d.sx[i], d.sw[i], d.so[i] = p["sx"][i], p["sw"][i], p["so"][i]
                d.combine, d.reduce, d.beta, d.beta_in_loop = p["combine"], p["reduce"], p["beta"], p["beta_in_loop"]
                d.n_epi = self._epi(slots, step, d.epi)
                descs.append((native.conv2d_nchw, d))
            else:
                d = native.NestDesc()
                d.n_out, d.n_red = p["n_out"], p["n_red"]
                for i, e in enumerate(p["extent"]):
                    d.extent[i] = e
                d.n_operands = len(p["operands"])
                for o, op in enumerate(p["operands"]):
                    no = d.operand[o]
                    no.ptr = self._ptr(slots, (op["ref"], 0))
                    no.addr.base = op["base"]
                    for i, c in enumerate(op["coeff"]):
                        no.addr.coeff[i] = c
                    no.n_guards = len(op["guards"])
                    for q, (gc, gco, gs) in enumerate(op["guards"]):
                        no.guard[q].base = gc
                        for i, c in enumerate(gco):
                            no.guard[q].coeff[i] = c
                        no.guard_size[q] = gs
                    no.fill = op["fill"]
                d.out = self._ptr(slots, (p["out"][0], 0))
                d.out_addr.base = p["out"][1]
                for i, c in enumerate(p["out_coeff"]):
                    d.out_addr.coeff[i] = c
                d.combine, d.reduce, d.beta = p["combine"], p["reduce"], p["beta"]
                d.n_epi = self._epi(slots, step, d.epi)
                descs.append((native.affine_nest, d))
        return descs

    def launch(self, slots: dict[int, int], stream: int = 0) -> int:
        """Enqueue every step on ``stream``; ``slots`` maps slot -> device ptr.
        Returns the number of kernel launches issued."""
        key = tuple(sorted(slots.items()))
        if key != self._desc_key:
            self._descs = self._build(slots)
            self._desc_key = key
        before = native.launch_count()
        for fn, d in self._descs:
            fn(d, stream)
        return native.launch_count() - before

    def launch_rows(self, slots: dict[int, int], stream: int, r0: int, r1: int,
                    b_unchanged: bool = False) -> int:
        """Rows [r0, r1) of a single-GEMM plan (row-block streaming)."""
        key = tuple(sorted(slots.items()))
        if key != self._desc_key:
            self._descs = self._build(slots)
            self._desc_key = key
        (fn, d), = self._descs
        blk = native.GemmDesc()
        ctypes.pointer(blk)[0] = d
        blk.m_begin, blk.m_end = r0, r1
        blk.flags = native.GEMM_B_UNCHANGED if b_unchanged else 0
        before = native.launch_count()
        fn(blk, stream)
        return native.launch_count() - before

    def descs(self, slots: dict[int, int]):
        key = tuple(sorted(slots.items()))
        if key != self._desc_key:
            self._descs = self._build(slots)
            self._desc_key = key
        return self._descs

    def launch_blocked(self, slots: dict[int, int], stream: int, flags: int, gen: int,
                       r0: int, r1: int, c0: int, c1: int) -> int:
        """One step of a blocked 3xTF32 sequence (lsb.h LSB_GEMM_PREP_A /
        PREP_B / PRESPLIT): split A rows [r0, r1) and/or B columns [c0, c1)
        into the resident split workspace, and/or compute the output
        rectangle rows [r0, r1) x columns [c0, c1) from what is split."""
        (fn, d), = self.descs(slots)
        blk = native.GemmDesc()
        ctypes.pointer(blk)[0] = d
        blk.m_begin, blk.m_end, blk.n_begin, blk.n_end = r0, r1, c0, c1
        blk.flags, blk.gen = flags, gen
        before = native.launch_count()
        fn(blk, stream)
        return native.launch_count() - before

    def streams(self):
        if not hasattr(self, "_streams"):
            self._streams = (native.Stream(), native.Stream(), native.Stream())
        return self._streams


def run_device(kernel: CompiledKernel, slots: dict[int, int], stream: int = 0) -> int:
    """Run on caller-owned device buffers (slot -> device pointer, e.g. torch
    ``data_ptr()``), inputs already resident; asynchronous on ``stream``.
    Output slots must point at buffers holding C_in when alpha != 0."""
    missing = set(kernel.slot_shapes) - set(slots)
    if missing:
        raise ShapeMismatch(f"slots {sorted(missing)} have no device buffer")
    return kernel.runner.launch(slots, stream)


#: host buffers at least this large that are not page-locked cross PCIe
#: through liblsb's staging slots (lsb_stage_*: pinned ring + host copy pool);
#: a plain pageable cudaMemcpyAsync runs at ~11 GB/s and blocks the caller
STAGE_MIN_BYTES = 1 << 20


def _pinned(arr) -> bool:
    return arr.nbytes < STAGE_MIN_BYTES or native.is_pinned(arr.ctypes.data)


def _h2d(dst: int, src: int, nbytes: int, stream: int, pinned: bool) -> None:
    if pinned:
        native.h2d(dst, src, nbytes, stream)
    else:
        native.stage_h2d_2d(dst, nbytes, src, nbytes, nbytes, 1, stream)


def _h2d_2d(dst, dpitch, src, spitch, width, height, stream, pinned) -> None:
    if pinned:
        native.h2d_2d(dst, dpitch, src, spitch, width, height, stream)
    else:
        native.stage_h2d_2d(dst, dpitch, src, spitch, width, height, stream)


def _d2h(dst: int, src: int, nbytes: int, stream: int, pinned: bool) -> None:
    if pinned:
        native.d2h(dst, src, nbytes, stream)
    else:
        native.stage_d2h_2d(dst, nbytes, src, nbytes, nbytes, 1, stream)


def _d2h_2d(dst, dpitch, src, spitch, width, height, stream, pinned) -> None:
    if pinned:
        native.d2h_2d(dst, dpitch, src, spitch, width, height, stream)
    else:
        native.stage_d2h_2d(dst, dpitch, src, spitch, width, height, stream)


def _reads_c_in(plan: Plan) -> bool:
    return any(e.c_in is not None for s in plan.steps for e in s.epi)


#: row-block streaming kicks in from this many multiply-adds (one launch
#: computes faster than its operands cross PCIe below it)
STREAM_MIN_MACS = 1 << 34
STREAM_BLOCKS = 8


def _row_stream_plan(kernel: CompiledKernel, hosts: dict):
    """Row blocks for copy/compute overlap, or None.  Applies to a plan that
    is one batch-1 GEMM whose A rows and C rows are contiguous byte ranges of
    their slots (M the slowest dim of both)."""
    plan = kernel.plan
    if len(plan.steps) != 1 or plan.steps[0].kind != "gemm":
        return None
    p = plan.steps[0].params
    if p["batch"] != 1 or p["M"] < 2 * STREAM_BLOCKS * 128 or p["M"] * p["N"] * p["K"] < STREAM_MIN_MACS:
        return None
    (aref, abase), (cref, cbase) = p["A"], p["C"]
    if aref.kind != "slot" or cref.kind != "slot" or abase or cbase:
        return None
    asize = int(np.prod(plan.slot_shapes[aref.key]))
    csize = int(np.prod(plan.slot_shapes[cref.key]))
    if p["sa_m"] * p["M"] != asize or p["sc_m"] * p["M"] != csize:
        return None
    if aref.key not in hosts:
        return None
    M = p["M"]
    per = -(-M // STREAM_BLOCKS)
    per = -(-per // 128) * 128
    return [(r0, min(M, r0 + per)) for r0 in range(0, M, per)], aref.key, cref.key, p["sa_m"], p["sc_m"]


def _execute_row_streamed(kernel, r: "Runner", dev, hosts, buffers, rows) -> int:
    """H2D of A row-block i+1 and D2H of C row-block i-1 overlap the
    contraction of block i (three streams; PCIe is full duplex).  B and the
    other operands go up once; the 3xTF32 path splits B once
    (LSB_GEMM_B_UNCHANGED on blocks after the first)."""
    blocks, a_slot, c_slot, sa_m, sc_m = rows
    s_in, s_c, s_out = r.streams()
    pre = native.Event()
    for slot, host in hosts.items():
        if slot not in (a_slot, c_slot):
            _h2d(dev[slot], host.ctypes.data, host.nbytes, s_in.handle, _pinned(host))
    pre.record(s_in)
    s_c.wait(pre)
    ahost = hosts[a_slot]
    chost_in = hosts.get(c_slot)       # C_in rows when the plan reads it
    dst = buffers.get(c_slot)
    direct = (dst is not None and dst.dtype == np.float32 and dst.flags.c_contiguous
              and dst.flags.writeable)
    out = dst if direct else np.empty(kernel.slot_shapes[c_slot], np.float32)
    a_pin, c_pin, o_pin = _pinned(ahost), chost_in is None or _pinned(chost_in), _pinned(out)
    launches = 0
    events = []
    for i, (r0, r1) in enumerate(blocks):
        ein, ec = native.Event(), native.Event()
        _h2d(dev[a_slot] + 4 * r0 * sa_m, ahost.ctypes.data + 4 * r0 * sa_m, 4 * (r1 - r0) * sa_m,
             s_in.handle, a_pin)
        if chost_in is not None:
            _h2d(dev[c_slot] + 4 * r0 * sc_m, chost_in.ctypes.data + 4 * r0 * sc_m,
                 4 * (r1 - r0) * sc_m, s_in.handle, c_pin)
        ein.record(s_in)
        s_c.wait(ein)
        launches += r.launch_rows(dev, s_c.handle, r0, r1, b_unchanged=i > 0)
        ec.record(s_c)
        s_out.wait(ec)
        _d2h(out.ctypes.data + 4 * r0 * sc_m, dev[c_slot] + 4 * r0 * sc_m, 4 * (r1 - r0) * sc_m,
             s_out.handle, o_pin)
        events.append((ein, ec))
    s_out.sync()
    s_c.sync()
    native.stage_wait()
    if not direct:
        if dst is not None:
            dst.reshape(-1)[:] = out.reshape(-1).astype(dst.dtype)
        else:
            buffers[c_slot] = out
    return launches


#: blocked tensor-core GEMM schedule.  Short reductions (K < 4096) are
#: download-bound: A row and B column pieces interleave, K/1024 clamped to
#: [4, 16] of each (C4: 4 pieces, 1.7 ms; 8 and 16 are no better).  Long
#: ones upload B whole first, then A in K/512 (<= 32) row pieces, each
#: computed as a full row strip as it lands: output (and its download) then
#: grows linearly instead of as the growing L of the interleaved order,
#: whose last L left ~3 ms of download after the compute (C5 e2e: 47.2 ms
#: interleaved, 44.8 B-first with 16 pieces, 44.1 with 32;
#: tools/dbg/e2e_order.py, tools/blocked_timeline.py).  Piece sizes are
#: multiples of 256 (the widest output tile).  BLOCK_PIECES overrides the
#: piece count.
BLOCK_PIECES = None
BLOCK_B_FIRST_K = 4096
_block_gen = [1 << 30]     # sequence ids, disjoint from the library's per-call stamps


def _blocked_plan(kernel: CompiledKernel, r: "Runner", dev, hosts: dict):
    """Blocked schedule for one fp32 (mul, add) GEMM on the 3xTF32 kernel whose
    A is [M][K] rows of its own slot, B is [K][N] or [N][K] in its own slot and
    C is [M][N] in its own slot with no C_in; else None."""
    plan = kernel.plan
    if os.environ.get("LSB_NO_BLOCKED") or len(plan.steps) != 1 or plan.steps[0].kind != "gemm":
        return None
    p = plan.steps[0].params
    M, N, K = p["M"], p["N"], p["K"]
    if p["batch"] != 1 or M * N * K < STREAM_MIN_MACS or _reads_c_in(plan):
        return None
    if M < 2 * 256 or N < 2 * 256:
        return None
    (aref, abase), (bref, bbase), (cref, cbase) = p["A"], p["B"], p["C"]
    if any(x.kind != "slot" for x in (aref, bref, cref)) or abase or bbase or cbase:
        return None
    if len({aref.key, bref.key, cref.key}) != 3 or aref.key not in hosts or bref.key not in hosts:
        return None
    size = lambda ref: int(np.prod(plan.slot_shapes[ref.key]))
    if not (p["sa_k"] == 1 and p["sa_m"] == K and size(aref) == M * K):
        return None
    if p["sb_n"] == 1 and p["sb_k"] == N and size(bref) == K * N:
        b_rowmajor = True          # [K][N]: column pieces are pitched copies
    elif p["sb_k"] == 1 and p["sb_n"] == K and size(bref) == K * N:
        b_rowmajor = False         # [N][K]: column pieces are contiguous
    else:
        return None
    if not (p["sc_n"] == 1 and p["sc_m"] == N and size(cref) == M * N):
        return None
    (_, d), = r.descs(dev)
    if native.gemm_algo(d) != "tf32x3":
        return None

    b_first = K >= BLOCK_B_FIRST_K
    npieces = BLOCK_PIECES or (max(4, min(32, K // 512)) if b_first else max(4, min(16, K // 1024)))

    def pieces(n):
        per = -(-(-(-n // npieces)) // 256) * 256
        return [(x, min(n, x + per)) for x in range(0, n, per)]
    return dict(M=M, N=N, K=K, a=aref.key, b=bref.key, c=cref.key, b_rowmajor=b_rowmajor,
                rows=pieces(M), cols=[(0, N)] if b_first else pieces(N))


def _execute_blocked(kernel, r: "Runner", dev, hosts, buffers, bp) -> int:
    """Copy/compute overlap over both operands: A row pieces and B column
    pieces cross PCIe interleaved (A0 B0 A1 B1 ...; for long reductions B is
    one piece, so the order is A0 B A1 A2 ...); each is split into the
    resident 3xTF32 workspace as it lands (PREP_A / PREP_B), and as soon as
    pieces i of A and B are both resident the new L of the output -- rows
    [0, i] x column piece i, then row piece i x columns [0, i) -- is computed
    (PRESPLIT) and its rectangles go back to the host as pitched copies while
    the next pieces upload.  Three streams; PCIe is full duplex."""
    M, N, K = bp["M"], bp["N"], bp["K"]
    a_slot, b_slot, c_slot = bp["a"], bp["b"], bp["c"]
    rows, cols = bp["rows"], bp["cols"]
    s_in, s_c, s_out = r.streams()
    for slot, host in hosts.items():
        if slot not in (a_slot, b_slot, c_slot):
            _h2d(dev[slot], host.ctypes.data, host.nbytes, s_in.handle, _pinned(host))
    ahost, bhost = hosts[a_slot], hosts[b_slot]
    dst = buffers.get(c_slot)
    direct = (dst is not None and dst.dtype == np.float32 and dst.flags.c_contiguous and dst.flags.writeable)
    out = dst if direct else np.empty(kernel.slot_shapes[c_slot], np.float32)
    a_pin, b_pin, o_pin = _pinned(ahost), _pinned(bhost), _pinned(out)
    _block_gen[0] = _block_gen[0] + 1 if _block_gen[0] < (1 << 31) - 2 else 1 << 30
    gen = _block_gen[0]
    PA, PB, PS = native.GEMM_PREP_A, native.GEMM_PREP_B, native.GEMM_PRESPLIT
    launches = 0
    keep = []
    nsteps = max(len(rows), len(cols))

    def d2h_rect(r0, r1, c0, c1):
        _d2h_2d(out.ctypes.data + 4 * (r0 * N + c0), 4 * N, dev[c_slot] + 4 * (r0 * N + c0), 4 * N,
                4 * (c1 - c0), r1 - r0, s_out.handle, o_pin)

    for i in range(nsteps):
        ea, eb = native.Event(), native.Event()
        if i < len(rows):
            r0, r1 = rows[i]
            _h2d(dev[a_slot] + 4 * r0 * K, ahost.ctypes.data + 4 * r0 * K, 4 * (r1 - r0) * K, s_in.handle, a_pin)
            ea.record(s_in)
        if i < len(cols):
            c0, c1 = cols[i]
            if bp["b_rowmajor"]:
                _h2d_2d(dev[b_slot] + 4 * c0, 4 * N, bhost.ctypes.data + 4 * c0, 4 * N, 4 * (c1 - c0), K,
                        s_in.handle, b_pin)
            else:
                _h2d(dev[b_slot] + 4 * c0 * K, bhost.ctypes.data + 4 * c0 * K, 4 * (c1 - c0) * K,
                     s_in.handle, b_pin)
            eb.record(s_in)
        if i < len(rows):
            s_c.wait(ea)
            launches += r.launch_blocked(dev, s_c.handle, PA, gen, rows[i][0], rows[i][1], 0, 0)
        if i < len(cols):
            s_c.wait(eb)
            launches += r.launch_blocked(dev, s_c.handle, PB, gen, 0, 0, cols[i][0], cols[i][1])
        # resident before / after this step: the new region is the L
        # [0, m1) x [0, n1) minus [0, m0) x [0, n0)
        m0 = rows[min(i, len(rows)) - 1][1] if i else 0
        n0 = cols[min(i, len(cols)) - 1][1] if i else 0
        m1, n1 = rows[min(i + 1, len(rows)) - 1][1], cols[min(i + 1, len(cols)) - 1][1]
        strips = [(0, m1, n0, n1), (m0, m1, 0, n0)]
        strips = [x for x in strips if x[1] > x[0] and x[3] > x[2]]
        if i < nsteps - 1:
            # one launch for the whole L (fewer partial waves), then its strips
            launches += r.launch_blocked(dev, s_c.handle, PS | native.GEMM_GROW, gen, m0, m1, n0, n1)
            ec = native.Event()
            ec.record(s_c)
            s_out.wait(ec)
            for x in strips:
                d2h_rect(*x)
            keep.append(ec)
        else:
            # the last L in halves of each strip, each copied back while the
            # next computes: the tail after the final upload is short
            for (r0, r1, c0, c1) in strips:
                if r1 - r0 >= c1 - c0:
                    mid = r0 + (r1 - r0) // 2 // 256 * 256
                    parts = [(r0, mid, c0, c1), (mid, r1, c0, c1)]
                else:
                    mid = c0 + (c1 - c0) // 2 // 256 * 256
                    parts = [(r0, r1, c0, mid), (r0, r1, mid, c1)]
                for x in parts:
                    if x[1] <= x[0] or x[3] <= x[2]:
                        continue
                    launches += r.launch_blocked(dev, s_c.handle, PS, gen, *x)
                    ec = native.Event()
                    ec.record(s_c)
                    s_out.wait(ec)
                    d2h_rect(*x)
                    keep.append(ec)
        keep += [ea, eb]
    s_out.sync()
    s_c.sync()
    native.stage_wait()
    if not direct:
        if dst is not None:
            dst.reshape(-1)[:] = out.reshape(-1).astype(dst.dtype)
        else:
            buffers[c_slot] = out
    return launches


def execute(kernel: CompiledKernel, buffers: dict[int, np.ndarray]) -> None:
    """Reference contract (backend.py:121-161): inputs required and never
    mutated, sizes checked (ShapeMismatch), a present output slot is read as
    C_in, outputs written in place (cast to the array's dtype) or inserted."""
    for slot in kernel.input_slots:
        if slot not in buffers:
            raise ShapeMismatch(f"input slot {slot} missing")
    for slot, shape in kernel.slot_shapes.items():
        if slot in buffers:
            want = int(np.prod(shape)) if shape else 1
            if buffers[slot].size != want:
                raise ShapeMismatch(f"slot {slot}: expected {shape} ({want} elems), "
                                    f"got {buffers[slot].size}")
    r = kernel.runner
    dev = r.slot_buffers()
    stream = 0
    staged = []
    hosts = {}
    for slot, arr in buffers.items():
        if slot in dev:
            hosts[slot] = np.ascontiguousarray(arr, dtype=np.float32)
    reads_cin = _reads_c_in(kernel.plan)
    for slot in kernel.output_slots:
        if slot not in buffers and reads_cin:
            # absent output read as C_in: zeros (the reference arena is np.zeros)
            n = int(np.prod(kernel.slot_shapes[slot])) if kernel.slot_shapes[slot] else 1
            hosts[slot] = np.zeros(n, np.float32)
    bp = _blocked_plan(kernel, r, dev, hosts)
    if bp is not None:
        launches = _execute_blocked(kernel, r, dev, hosts, buffers, bp)
        kernel._count(launches)
        return
    rows = _row_stream_plan(kernel, hosts)
    if rows is not None:
        launches = _execute_row_streamed(kernel, r, dev, hosts, buffers, rows)
        kernel._count(launches)
        return
    for slot, host in hosts.items():
        staged.append(host)
        _h2d(dev[slot], host.ctypes.data, host.nbytes, stream, _pinned(host))
    launches = r.launch(dev, stream)
    outs = {}
    for slot in kernel.output_slots:
        dst = buffers.get(slot)
        if (dst is not None and dst.dtype == np.float32 and dst.flags.c_contiguous
                and dst.flags.writeable):
            # straight into the caller's array (pinned: one DMA; pageable:
            # through the staging slots)
            _d2h(dst.ctypes.data, dev[slot], dst.nbytes, stream, _pinned(dst))
            continue
        res = np.empty(kernel.slot_shapes[slot], np.float32)
        _d2h(res.ctypes.data, dev[slot], res.nbytes, stream, _pinned(res))
        outs[slot] = res
    native.sync(stream)
    native.stage_wait()
    del staged
    kernel._count(launches)
    for slot, res in outs.items():
        if slot in buffers:
            dst = buffers[slot]
            dst.reshape(-1)[:] = res.reshape(-1).astype(dst.dtype)
        else:
            buffers[slot] = res
