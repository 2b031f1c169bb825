"""Plan a loopsmith dataflow graph onto the B200 kernel set.

The reference lowers a graph to a loop tree and emits one flat VM program
(backend.py:1427-1454).  Results are schedule-independent by construction
(feedback.py:69-75: the oracle ignores every schedule annotation), so this
planner works from the graph's arithmetic and uses the schedule only as a
tile hint.  It cuts the graph into *groups*, one kernel launch each:

  contraction group   [combine node] -> reduce node -> elementwise chain
                      (bias add, ReLU, sigmoid, alpha*pre(C_in) ...), the
                      chain fused into the epilogue (lsb_epi_stage) so the
                      intermediate never round-trips HBM (backend.py:544-548,
                      1301-1310 keep it in registers for the same reason);
  copy group          a Write fed by a Read/View (transpose, slice, concat).

Each group maps to the first kernel whose contract it satisfies:

  lsb_semiring_gemm   2 operands, unguarded affine access, every index group
                      (batch / M / N / K) flattenable to one stride per tensor
  lsb_conv2d_nchw     (mul, add) over a 4-D windowed View  (NCHW conv, guarded
                      views = padding with the view's oob)
  lsb_affine_nest     anything else (any views, guards, operand count <= 4)

Unsupported graphs raise ``BlockTooLarge`` (the reference's "cannot express"
error, backend.py:41-42) -- never a CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from .errors import BlockTooLarge
from .graph import EW_CODE, OP_CODE, Graph, GNode
from .schedule import read_schedule

MAX_EPI = 4
MAX_NEST_DIMS = 8
MAX_NEST_OPERANDS = 4
MAX_GUARDS = 4


# ---------------------------------------------------------------------------
# buffers and affine accesses
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Ref:
    """A device buffer: an external slot or a scratch intermediate."""
    kind: str   # "slot" | "scratch"
    key: int


@dataclass
class Access:
    """element = buf[base + Σ coeff[v] * iter(v)]; guarded coordinates
    (const + Σ c[v] * iter(v) outside [0, size)) read ``fill``."""
    ref: Ref
    base: int
    coeff: dict[int, int]
    guards: list[tuple[int, dict[int, int], int]] = field(default_factory=list)
    fill: float = 0.0

    def c(self, v: int) -> int:
        return self.coeff.get(v, 0)


@dataclass
class EpiSpec:
    combine: int = -1
    reduce: int = 0
    pre: int = 0
    post: int = 0
    beta: float = 1.0
    alpha: float = 0.0
    operand: Optional[Access] = None
    c_in: Optional[Access] = None


@dataclass
class Step:
    kind: str                    # "gemm" | "conv" | "nest"
    nodes: list[int]             # graph nodes this launch evaluates
    params: dict
    epi: list[EpiSpec]
    flops: int = 0

    def describe(self) -> str:
        p = self.params
        if self.kind == "gemm":
            return (f"gemm[{p['combine_name']},{p['reduce_name']}] batch={p['batch']} "
                    f"M={p['M']} N={p['N']} K={p['K']} epi={len(self.epi)} nodes={self.nodes}")
        if self.kind == "conv":
            return (f"conv[n={p['N']} c={p['C']} {p['H']}x{p['W']} co={p['CO']} "
                    f"{p['R']}x{p['S']} s={p['stride_h']} pad={p['pad_h']}] nodes={self.nodes}")
        return (f"nest[{p['combine_name']},{p['reduce_name']}] out={p['extent'][:p['n_out']]} "
                f"red={p['extent'][p['n_out']:]} ops={len(p['operands'])} nodes={self.nodes}")


@dataclass
class Plan:
    graph: Graph
    steps: list[Step]
    slot_shapes: dict[int, tuple[int, ...]]
    input_slots: set[int]
    output_slots: set[int]
    scratch: dict[int, int]      # scratch key (node id) -> elements

    @property
    def scratch_bytes(self) -> int:
        return 4 * sum(self.scratch.values())

    def describe(self) -> str:
        return "\n".join(s.describe() for s in self.steps) + "\n"


def _row_major(sizes: list[int]) -> list[int]:
    strides, acc = [], 1
    for s in reversed(sizes):
        strides.append(acc)
        acc *= s
    return strides[::-1]


# ---------------------------------------------------------------------------
# the planner
# ---------------------------------------------------------------------------

class Planner:
    def __init__(self, graph: Graph):
        self.g = graph
        self.slot_shapes = graph.slot_shapes()
        self.scratch: dict[int, int] = {}
        self.home: dict[int, tuple[Ref, dict[int, int]]] = {}   # node -> (buffer, var strides)
        self.steps: list[Step] = []
        self._operand_nodes: list[int] = []

    # ---- where a node's value lives ----------------------------------------

    def _slot_strides(self, node: GNode) -> dict[int, int]:
        st = _row_major([self.g.size(d) for d in node.dims])
        return {d: s for d, s in zip(node.dims, st)}

    def _materialize_home(self, node: GNode) -> tuple[Ref, dict[int, int]]:
        """A group's output: its Write slot if it has one, else scratch."""
        w = self.g.write_of(node.id)
        if w is not None:
            # the slot layout is the write node's dims (frontend.py:128-138)
            return Ref("slot", w.slot), self._slot_strides(w)
        self.scratch[node.id] = max(1, self._elems(node))
        return Ref("scratch", node.id), self._slot_strides(node)

    def _elems(self, node: GNode) -> int:
        n = 1
        for d in node.dims:
            n *= self.g.size(d)
        return n

    def access(self, nid: int) -> Access:
        """Affine access of node ``nid``'s value indexed by its own dims."""
        node = self.g[nid]
        if node.kind == "read":
            return Access(Ref("slot", node.slot), 0, self._slot_strides(node))
        if nid in self.home:
            ref, strides = self.home[nid]
            return Access(ref, 0, dict(strides))
        if node.kind == "view":
            src = self.access(node.inputs[0])
            if src.guards:
                raise BlockTooLarge(f"view {nid} over a guarded view is not composed")
            srcnode = self.g[node.inputs[0]]
            base = src.base
            coeff: dict[int, int] = {}
            guards = []
            for c in node.constraints:
                stride = src.c(c.input_dim)
                if c.input_dim not in srcnode.dims:
                    raise BlockTooLarge(f"view {nid}: constraint on unknown dim")
                base += stride * c.offset
                for v, co in c.terms:
                    coeff[v] = coeff.get(v, 0) + stride * co
                if node.guarded:
                    guards.append((c.offset, {v: co for v, co in c.terms}, self.g.size(c.input_dim)))
            # dims of the source not constrained cannot exist (validate: view-unconstrained-input-dim)
            return Access(src.ref, base, {v: x for v, x in coeff.items() if x}, guards,
                          node.oob if node.guarded else 0.0)
        raise BlockTooLarge(f"node {nid} ({node.kind}) has no materialized value")

    # ---- grouping -----------------------------------------------------------

    def _absorbable_combine(self, r: GNode) -> Optional[GNode]:
        if len(r.inputs) != 1:
            return None
        p = self.g[r.inputs[0]]
        if (p.kind == "arith" and len(p.inputs) >= 2 and not self.g.reduction_dims(p)
                and p.pre == "identity" and p.post == "identity" and p.alpha == 0.0
                and p.beta == 1.0 and len(self.g.consumers(p.id)) == 1
                and p.id not in self.home):
            return p
        return None

    def _next_epilogue(self, tail: GNode, out_dims: set[int]) -> Optional[GNode]:
        cons = self.g.consumers(tail.id)
        if len(cons) != 1:
            return None
        e = cons[0]
        if e.kind != "arith" or self.g.reduction_dims(e) or set(e.dims) != out_dims:
            return None
        others = [i for i in e.inputs if i != tail.id]
        if e.inputs.count(tail.id) != 1 or len(others) > 1:
            return None
        for o in others:
            on = self.g[o]
            if on.kind not in ("read", "view") and o not in self.home:
                return None
            if not set(on.dims) <= out_dims:
                return None
        return e

    def plan(self) -> Plan:
        g = self.g
        done: set[int] = set()
        for nid in g.topo_order():
            node = g[nid]
            if nid in done or node.kind in ("read", "view"):
                continue
            if node.kind == "write":
                src = g[node.inputs[0]]
                home = self.home.get(src.id)
                if src.kind in ("read", "view") or (home and home[0] != Ref("slot", node.slot)):
                    self._copy_step(node)
                continue
            # arith: group head?  (a combine node absorbed by its consumer is
            # planned with the consumer)
            cons = g.consumers(nid)
            if (len(cons) == 1 and cons[0].kind == "arith" and g.reduction_dims(cons[0])
                    and self._absorbable_combine(cons[0]) is node):
                continue
            self._contraction_group(node, done)
        return Plan(g, self.steps, self.slot_shapes, g.input_slots(), g.output_slots(),
                    dict(self.scratch))

    def _contraction_group(self, r: GNode, done: set[int]) -> None:
        g = self.g
        comb_node = self._absorbable_combine(r) if g.reduction_dims(r) else None
        if comb_node is not None:
            operands = list(comb_node.inputs)
            combine = comb_node.combine_op
            nodes = [comb_node.id, r.id]
        else:
            operands = list(r.inputs)
            combine = r.combine_op
            nodes = [r.id]
        if len(operands) > MAX_NEST_OPERANDS:
            raise BlockTooLarge(f"node {r.id}: {len(operands)} operands")
        out_dims = set(r.dims)
        chain: list[GNode] = []
        tail = r
        while len(chain) + 1 < MAX_EPI and g.write_of(tail.id) is None:
            e = self._next_epilogue(tail, out_dims)
            if e is None:
                break
            chain.append(e)
            tail = e
        nodes += [e.id for e in chain]
        done.update(nodes)

        home_ref, home_strides = self._materialize_home(tail)
        out = Access(home_ref, 0, dict(home_strides))
        write = g.write_of(tail.id)

        red = g.reduction_dims(r)
        # stage 0: the contraction node itself
        def cin_access(node: GNode) -> Access:
            w = g.write_of(node.id)
            if w is None:
                raise BlockTooLarge(f"node {node.id} has alpha != 0 but no write consumer")
            return Access(Ref("slot", w.slot), 0, self._slot_strides(w))

        epi: list[EpiSpec] = []
        s0 = EpiSpec(reduce=OP_CODE[r.reduce_op], pre=EW_CODE[r.pre], post=EW_CODE[r.post],
                     alpha=r.alpha)
        if r.alpha != 0.0:
            s0.c_in = cin_access(r)
        epi.append(s0)
        prev = r
        for e in chain:
            st = EpiSpec(reduce=OP_CODE[e.reduce_op], pre=EW_CODE[e.pre], post=EW_CODE[e.post],
                         beta=e.beta, alpha=e.alpha)
            others = [i for i in e.inputs if i != prev.id]
            if others:
                st.combine = OP_CODE[e.combine_op]
                st.operand = self.access(others[0])
                if st.operand.guards:
                    raise BlockTooLarge(f"node {e.id}: guarded epilogue operand")
            if e.alpha != 0.0:
                st.c_in = cin_access(e)
            epi.append(st)
            prev = e

        accesses = [self.access(o) for o in operands]
        self._operand_nodes = list(operands)
        beta = r.beta
        redop = r.reduce_op
        out_vars = list(r.dims)

        step = None
        if red and len(accesses) == 2:
            step = self._try_gemm(r, nodes, accesses, out, out_vars, red, combine, redop, beta, epi)
            if step is None and combine == "mul" and redop == "add":
                step = self._try_conv(r, nodes, operands, accesses, out, out_vars, red, beta, epi)
        if step is None:
            step = self._nest(r, nodes, accesses, out, out_vars, red, combine, redop, beta, epi)
        self.steps.append(step)
        self.home[tail.id] = (home_ref, home_strides)
        del write

    # ---- kernel matching ----------------------------------------------------

    @staticmethod
    def _beta_plan(combine: str, redop: str, beta: float):
        """Where beta goes: (kernel_reduce, beta_in_loop, post_scale).
        Tuned kernels have no per-term beta; move it out only when that is
        exact (max/min: monotone scaling) or within fp32 tolerance (add)."""
        tuned = (combine, redop) in (("mul", "add"), ("add", "max"), ("add", "min"))
        if beta == 1.0:
            return redop, not tuned, 1.0
        if tuned and redop == "add":
            return redop, False, beta
        if tuned and redop in ("max", "min") and beta > 0:
            return redop, False, beta
        if tuned and redop in ("max", "min") and beta < 0:
            return ("min" if redop == "max" else "max"), False, beta
        return redop, True, 1.0

    def _flatten(self, group: list[int], tensors: list[Access], order_key) -> Optional[tuple]:
        """Flatten index vars into one index; returns (extent, [stride per tensor])."""
        if not group:
            return 1, [0] * len(tensors)
        vs = sorted(group, key=order_key)
        ext = 1
        for v in vs:
            ext *= self.g.size(v)
        strides = []
        for t in tensors:
            inner = vs[-1]
            unit = t.c(inner)
            acc = self.g.size(inner)
            for v in reversed(vs[:-1]):
                if t.c(v) != unit * acc:
                    return None
                acc *= self.g.size(v)
            strides.append(unit)
        return ext, strides

    def _try_gemm(self, r, nodes, acc, out, out_vars, red, combine, redop, beta, epi):
        if any(a.guards for a in acc):
            return None
        A, B = acc

        def classify(A, B):
            Mv, Nv, Bv = [], [], []
            for v in out_vars:
                ca, cb = A.c(v) != 0, B.c(v) != 0
                if ca and cb:
                    Bv.append(v)
                elif ca:
                    Mv.append(v)
                else:
                    Nv.append(v)     # B-only, or carried by neither (broadcast)
            return Mv, Nv, Bv

        Mv, Nv, Bv = classify(A, B)
        # the output's unit-stride var should land in N (coalesced stores)
        unit = [v for v in out_vars if out.c(v) == 1]
        if unit and unit[0] in Mv:
            A, B = B, A
            Mv, Nv, Bv = classify(A, B)
        epi_ops = [e.operand for e in epi if e.operand is not None] + \
                  [e.c_in for e in epi if e.c_in is not None]
        bykey = lambda t: (lambda v: -abs(t.c(v)))  # noqa: E731
        fm = self._flatten(Mv, [A, out] + epi_ops, bykey(out))
        fn = self._flatten(Nv, [B, out] + epi_ops, bykey(out))
        fb = self._flatten(Bv, [A, B, out] + epi_ops, bykey(out))
        fk = self._flatten(red, [A, B], bykey(A) if any(A.c(v) for v in red) else bykey(B))
        if None in (fm, fn, fb, fk):
            return None
        M, (sa_m, sc_m, *em) = fm
        N, (sb_n, sc_n, *en) = fn
        batch, (sa_b, sb_b, sc_b, *eb) = fb
        K, (sa_k, sb_k) = fk
        kred, in_loop, post_scale = self._beta_plan(combine, redop, beta)
        epi = [EpiSpec(**vars(e)) for e in epi]
        epi[0].beta = post_scale
        # per-stage operand strides in (batch, m, n) coordinates; epi_ops
        # lists operands first, then c_ins
        k_ops = sum(1 for e in epi if e.operand is not None)
        strides = []
        io, ic = 0, k_ops
        for e in epi:
            ent = {}
            if e.operand is not None:
                ent["operand"] = (eb[io], em[io], en[io], 0)
                io += 1
            if e.c_in is not None:
                ent["c_in"] = (eb[ic], em[ic], en[ic], 0)
                ic += 1
            strides.append(ent)
        # the schedule picks the launch configuration (schedule.py): register
        # block -> tile class, an outermost reduction loop -> split-K
        sched = read_schedule(self.g, r, Mv, Nv, list(red),
                              [o for o in (self._operand_nodes or [])])
        hints = sched.tile_hints()
        params = dict(M=M, N=N, K=K, batch=batch,
                      A=(A.ref, A.base), sa_b=sa_b, sa_m=sa_m, sa_k=sa_k,
                      B=(B.ref, B.base), sb_b=sb_b, sb_k=sb_k, sb_n=sb_n,
                      C=(out.ref, out.base), sc_b=sc_b, sc_m=sc_m, sc_n=sc_n,
                      combine=OP_CODE[combine], reduce=OP_CODE[kred],
                      combine_name=combine, reduce_name=kred,
                      beta=beta if in_loop else 1.0, beta_in_loop=int(in_loop),
                      epi_strides=strides, tile_m=hints["tile_m"], tile_n=hints["tile_n"],
                      split_k=hints["split_k"], schedule=sched)
        flops = 2 * M * N * K * batch
        return Step("gemm", nodes, params, epi, flops)

    def _try_conv(self, r, nodes, operands, acc, out, out_vars, red, beta, epi):
        g = self.g
        # identify the windowed operand: a View over a 4-D buffer
        for xi in (0, 1):
            xnode = g[operands[xi]]
            wacc = acc[1 - xi]
            if xnode.kind != "view" or len(xnode.constraints) != 4 or wacc.guards:
                continue
            src = g[xnode.inputs[0]]
            srcacc = self.access(src.id)
            if srcacc.guards:
                continue
            singles, windows = [], []
            for c in xnode.constraints:
                if len(c.terms) == 1 and c.terms[0][1] == 1:
                    singles.append(c)
                elif len(c.terms) == 2:
                    windows.append(c)
            if len(singles) != 2 or len(windows) != 2:
                continue
            outs, reds = set(out_vars), set(red)
            nc = [c for c in singles if c.terms[0][0] in outs]
            cc = [c for c in singles if c.terms[0][0] in reds]
            if len(nc) != 1 or len(cc) != 1:
                continue
            nvar, cvar = nc[0].terms[0][0], cc[0].terms[0][0]
            sp = []
            ok = True
            for c in windows:
                (v1, c1), (v2, c2) = c.terms
                if v1 in outs and v2 in reds:
                    sp.append((c, v1, c1, v2, c2))
                elif v2 in outs and v1 in reds:
                    sp.append((c, v2, c2, v1, c1))
                else:
                    ok = False
            if not ok:
                continue
            (ch, hvar, sh, rvar, dh), (cw, wvar, sw, svar, dw) = sp
            covars = [v for v in out_vars if v not in (nvar, hvar, wvar)]
            if len(covars) != 1 or set(red) != {cvar, rvar, svar}:
                continue
            co = covars[0]
            if any(wacc.c(v) for v in (nvar, hvar, wvar)):
                continue
            # weights must depend on exactly (co, c, r, s)
            sx = [srcacc.c(nc[0].input_dim), srcacc.c(cc[0].input_dim),
                  srcacc.c(ch.input_dim), srcacc.c(cw.input_dim)]
            if xnode.guarded:
                fill = xnode.oob
            else:
                fill = 0.0
            # non-zero offsets on the batch/channel coordinates shift the base
            xbase = srcacc.base + srcacc.c(nc[0].input_dim) * nc[0].offset + \
                srcacc.c(cc[0].input_dim) * cc[0].offset
            kred, in_loop, post_scale = self._beta_plan("mul", "add", beta)
            epi2 = [EpiSpec(**vars(e)) for e in epi]
            epi2[0].beta = post_scale
            strides = []
            for e in epi2:
                ent = {}
                if e.operand is not None:
                    ent["operand"] = tuple(e.operand.c(v) for v in (nvar, co, hvar, wvar))
                    # operands may only depend on the output coordinates
                if e.c_in is not None:
                    ent["c_in"] = tuple(e.c_in.c(v) for v in (nvar, co, hvar, wvar))
                strides.append(ent)
            params = dict(N=g.size(nvar), C=g.size(cvar), H=g.size(ch.input_dim), W=g.size(cw.input_dim),
                          CO=g.size(co), R=g.size(rvar), S=g.size(svar),
                          HO=g.size(hvar), WO=g.size(wvar),
                          stride_h=sh, stride_w=sw, pad_h=-ch.offset, pad_w=-cw.offset,
                          dil_h=dh, dil_w=dw, fill=fill,
                          x=(srcacc.ref, xbase), sx=tuple(sx),
                          w=(wacc.ref, wacc.base), sw=tuple(wacc.c(v) for v in (co, cvar, rvar, svar)),
                          o=(out.ref, out.base), so=tuple(out.c(v) for v in (nvar, co, hvar, wvar)),
                          combine=OP_CODE["mul"], reduce=OP_CODE["add"],
                          beta=1.0, beta_in_loop=0, epi_strides=strides)
            if in_loop:
                return None
            flops = 2 * g.size(nvar) * g.size(co) * g.size(hvar) * g.size(wvar) * \
                g.size(cvar) * g.size(rvar) * g.size(svar)
            return Step("conv", nodes, params, epi2, flops)
        return None

    def _nest(self, r, nodes, acc, out, out_vars, red, combine, redop, beta, epi):
        dims = list(out_vars) + list(red)
        if len(dims) > MAX_NEST_DIMS:
            raise BlockTooLarge(f"node {r.id}: {len(dims)} loop dims exceed {MAX_NEST_DIMS}")
        ops = []
        for a in acc:
            if len(a.guards) > MAX_GUARDS:
                raise BlockTooLarge(f"node {r.id}: too many guarded coordinates")
            ops.append(dict(ref=a.ref, base=a.base, coeff=[a.c(v) for v in dims],
                            guards=[(gc, [gt.get(v, 0) for v in dims], gs) for gc, gt, gs in a.guards],
                            fill=a.fill))
        strides = []
        c4 = list(out_vars[:4])
        if len(out_vars) > 4:
            for e in epi:
                for acc_ in (e.operand, e.c_in):
                    if acc_ is not None and any(acc_.c(v) for v in out_vars[4:]):
                        raise BlockTooLarge(f"node {r.id}: epilogue over > 4 output dims")
        for e in epi:
            ent = {}
            if e.operand is not None:
                ent["operand"] = tuple([e.operand.c(v) for v in c4] + [0] * (4 - len(c4)))
            if e.c_in is not None:
                ent["c_in"] = tuple([e.c_in.c(v) for v in c4] + [0] * (4 - len(c4)))
            strides.append(ent)
        params = dict(n_out=len(out_vars), n_red=len(red),
                      extent=[self.g.size(v) for v in dims],
                      operands=ops, out=(out.ref, out.base),
                      out_coeff=[out.c(v) for v in out_vars] + [0] * len(red),
                      combine=OP_CODE[combine], reduce=OP_CODE[redop],
                      combine_name=combine, reduce_name=redop,
                      beta=beta, epi_strides=strides)
        pts = 1
        for v in dims:
            pts *= self.g.size(v)
        return Step("nest", nodes, params, [EpiSpec(**vars(e)) for e in epi], 2 * pts)

    def _copy_step(self, w: GNode) -> None:
        """Write fed directly by a Read / View: a data-movement nest."""
        src = self.access(w.inputs[0])
        out = Access(Ref("slot", w.slot), 0, self._slot_strides(w))
        dims = list(w.dims)
        if len(dims) > MAX_NEST_DIMS:
            raise BlockTooLarge(f"write {w.id}: {len(dims)} dims")
        if len(src.guards) > MAX_GUARDS:
            raise BlockTooLarge(f"write {w.id}: too many guards")
        ops = [dict(ref=src.ref, base=src.base, coeff=[src.c(v) for v in dims],
                    guards=[(gc, [gt.get(v, 0) for v in dims], gs) for gc, gt, gs in src.guards],
                    fill=src.fill)]
        params = dict(n_out=len(dims), n_red=0, extent=[self.g.size(v) for v in dims],
                      operands=ops, out=(out.ref, out.base),
                      out_coeff=[out.c(v) for v in dims],
                      combine=OP_CODE["add"], reduce=OP_CODE["add"],
                      combine_name="copy", reduce_name="-", beta=1.0, epi_strides=[])
        self.steps.append(Step("nest", [w.id], params, [], 0))


def plan_graph(graph) -> Plan:
    return Planner(Graph.coerce(graph)).plan()
