"""From a loopsmith schedule to B200 launch choices and modeled counters.

The reference compiles a scheduled loop tree into register-blocked vector
code (backend.py:593-691 ``_select_region``: the loops inside the innermost
reduction loop form the register block, capped at ``vregs - 8`` vector
registers) and counts the VM's memory instructions (program.py:186-190).
Results never depend on the schedule (feedback.py:69-75), so on the B200
the schedule chooses *how* a contraction runs:

* register block -> CTA tile class.  A block of at least 64 output elements
  (the BASELINE schedules' 4 x 64) keeps the kernel set's best tiles; a
  smaller block selects the 64-row SIMT tile and the 128-wide 3xTF32 tile
  (csrc/lsb_api.cu reads ``tile_m`` / ``tile_n``);
* a reduction loop outside every output loop (``k_o`` outermost) asks for
  split-K with that many slices (SIMT kernel, ``split_k``, capped at 16);
* a staged Read (``schedule.stage``) is a smem-staged operand panel: the
  kernels stage every operand through shared memory, and the panel's size
  (the reference's ``Alloc.size``) is reported in ``scratch_bytes``.

``schedule_counters`` models the schedule's memory instructions the way the
reference VM counts them -- vector loads of the B panel and broadcasts of A
per reduction step of each register block, one store per output vector --
at the B200 kernels' 16-byte access width.  ``memory_access_count()`` and
the tuner's score (tuner.py:66-69) read it, so ``tune`` ranks schedules by
locality as it does on the CPU backend; measured time is in ``benchmark``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from .graph import Graph, GNode

#: 16-byte vectors of fp32 (the kernels' global / shared access width)
LANES = 4
#: register-block cap of the reference's avx512 preset (32 vregs - 8) x 16 lanes
MAX_BLOCK = 24 * 16
#: a block this large keeps the default (best measured) tiles
LARGE_BLOCK = 64
MAX_SPLIT_K = 16


@dataclass
class ScheduleMap:
    node: int                      # the contraction node the schedule is read from
    order: list[int]               # its loop vars, outermost first
    m_block: int = 1               # register block extent along M / N
    n_block: int = 1
    k_split: int = 1               # split-K slices requested (reduction loop outermost)
    raster_n: bool = False         # outermost output loop runs along N
    staged: list[tuple[int, int]] = field(default_factory=list)   # (read node, staging var)

    @property
    def block(self) -> int:
        return self.m_block * self.n_block

    def tile_hints(self) -> dict:
        """Launch hints for lsb_gemm_desc: tile_m / tile_n (0 = auto)."""
        small = self.block < LARGE_BLOCK
        return {"tile_m": 64 if small else 0, "tile_n": 128 if small else 0,
                "split_k": self.k_split if self.k_split > 1 else 0}

    def describe(self) -> str:
        s = f"block {self.m_block}x{self.n_block}"
        if self.k_split > 1:
            s += f", split-K {self.k_split}"
        if self.raster_n:
            s += ", N-major raster"
        if self.staged:
            s += f", {len(self.staged)} staged panel(s)"
        return s


def base_var(g: Graph, vid: int) -> int:
    while g.vars[vid].origin is not None:
        vid = g.vars[vid].origin[0]
    return vid


def read_schedule(g: Graph, node: GNode, m_vars: list[int], n_vars: list[int],
                  k_vars: list[int], operands: list[int]) -> ScheduleMap:
    """Schedule of contraction ``node`` (the reducing Arith node): M / N /
    K classes are base vars; the loop order is the node's own (leaf vars)."""
    order = list(node.order)
    cls = {}
    for v in order:
        b = base_var(g, v)
        cls[v] = "m" if b in m_vars else "n" if b in n_vars else "k" if b in k_vars else "?"
    sm = ScheduleMap(node.id, order)
    # register block: output loops inside the innermost reduction loop,
    # from the innermost outward while the block fits MAX_BLOCK elements
    last_k = max((i for i, v in enumerate(order) if cls[v] == "k"), default=-1)
    mb = nb = 1
    for v in reversed(order[last_k + 1:]):
        size = g.size(v)
        if cls[v] == "m" and mb * size * nb <= MAX_BLOCK:
            mb *= size
        elif cls[v] == "n" and mb * nb * size <= MAX_BLOCK:
            nb *= size
        else:
            break
    sm.m_block, sm.n_block = mb, nb
    # split-K: reduction loops outside every output loop
    first_out = min((i for i, v in enumerate(order) if cls[v] in ("m", "n")), default=len(order))
    ks = 1
    for v in order[:first_out]:
        if cls[v] == "k":
            ks *= g.size(v)
    sm.k_split = min(ks, MAX_SPLIT_K) if ks > 1 else 1
    outs = [v for v in order if cls[v] in ("m", "n")]
    sm.raster_n = bool(outs) and cls[outs[0]] == "n"
    for o in operands:
        on = g[o]
        if on.kind in ("read", "view") and on.staged:
            sm.staged.append((o, on.staged[0]))
    return sm


def schedule_counters(sm: ScheduleMap, M: int, N: int, K: int, batch: int = 1) -> tuple[int, int, int]:
    """(vload, vbroadcast, vstore) of the schedule as register-blocked code:
    per reduction step of an m_block x n_block block, n_block / 4 vector
    loads of B and m_block broadcasts of A; one store per output vector."""
    mb, nb = min(sm.m_block, M), min(sm.n_block, N)
    blocks = batch * -(-M // mb) * -(-N // nb)
    nvec = -(-nb // LANES)
    return blocks * K * nvec, blocks * K * mb, batch * M * -(-N // LANES)


def alloc_scratch_bytes(tree) -> Optional[int]:
    """scratch_bytes of a lowered tree by the reference's rule
    (backend.py:308-319): every non-Write allocation, except unstaged Reads
    and Views (consumers address their source directly), 4 bytes an element."""
    allocs = getattr(tree, "alloc", None)
    dfg = getattr(tree, "dfg", None)
    if allocs is None or dfg is None:
        return None
    total = 0
    for nid, alloc in allocs.items():
        node = dfg[nid]
        kind = type(node.kind).__name__.lower()
        if kind == "write":
            continue
        if kind in ("read", "view") and not node.staged:
            continue
        total += 4 * int(alloc.size)
    return total
