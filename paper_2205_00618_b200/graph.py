"""Neutral, read-only mirror of a loopsmith dataflow graph.

The B200 backend never imports the reference at run time: the GPU box has no
copy of it.  Instead it works on this small mirror, which can be built either
from a live ``loopsmith.ir.DFG`` (duck-typed attribute reads, here in the dev
container and in user processes that have loopsmith installed) or from the
reference's canonical graph JSON (``loopsmith.serialize.dfg_to_json``,
reference ``pkg/src/loopsmith/serialize.py:32-87``), which is how the parity
fixtures travel to the GPU box.

Semantics mirrored (reference file:line):
  * node kinds Read / Write / Arith / View           ir.py:168-245
  * Arith op -> (combine, reduce) pair, identities   ir.py:178-191
  * reduction_dims / iteration_dims                  ir.py:321-336
  * split lineage: expansion / padded_extent         ir.py:294-319
  * topo_order (Kahn, min-heap on node id)           ir.py:349-369
  * slot_shapes                                      feedback.py:46-52
"""

from __future__ import annotations

import heapq
import json
from dataclasses import dataclass, field
from typing import Optional

#: reference ir.py:182 OP_IDENTITY
OP_IDENTITY = {"add": 0.0, "mul": 1.0, "max": float("-inf"), "min": float("inf")}
#: reference ir.py:185-191 OP_SEMANTICS: node op -> (combine, reduce)
OP_SEMANTICS = {
    "add": ("add", "add"),
    "mul": ("mul", "mul"),
    "max": ("max", "max"),
    "min": ("min", "min"),
    "fma": ("mul", "add"),
}
#: reference ir.py:179 ELEMENTWISE_OPS
ELEMENTWISE_OPS = ("identity", "relu", "sigmoid")
#: numeric codes shared with the C-ABI; equal to program.py:182-183
#: KIND_CODE / EW_CODE so the two vocabularies never drift.
OP_CODE = {"add": 0, "mul": 1, "max": 2, "min": 3}
EW_CODE = {"identity": 0, "relu": 1, "sigmoid": 2}


class GraphError(Exception):
    """The graph (or its JSON) is malformed."""


@dataclass
class GVar:
    id: int
    name: str
    size: int
    origin: Optional[tuple[int, int, str]] = None  # (parent id, factor, part)


@dataclass
class GConstraint:
    input_dim: int
    terms: tuple[tuple[int, int], ...]  # (var id, coeff)
    offset: int = 0


@dataclass
class GNode:
    id: int
    kind: str                 # read | write | arith | view
    name: str
    inputs: tuple[int, ...]
    dims: tuple[int, ...]     # output buffer dims (var ids), row-major
    order: tuple[int, ...] = ()
    staged: tuple[int, ...] = ()
    slot: Optional[int] = None
    op: str = ""
    pre: str = "identity"
    post: str = "identity"
    alpha: float = 0.0
    beta: float = 1.0
    constraints: tuple[GConstraint, ...] = ()
    guarded: bool = False
    oob: float = 0.0

    @property
    def combine_op(self) -> str:
        return OP_SEMANTICS[self.op][0]

    @property
    def reduce_op(self) -> str:
        return OP_SEMANTICS[self.op][1]


@dataclass
class Graph:
    vars: dict[int, GVar] = field(default_factory=dict)
    nodes: dict[int, GNode] = field(default_factory=dict)

    # ---- construction -----------------------------------------------------

    @classmethod
    def from_json(cls, obj) -> "Graph":
        """Parse the reference's canonical graph JSON (serialize.py:32-87)."""
        if isinstance(obj, (str, bytes)):
            obj = json.loads(obj)
        g = cls()
        try:
            for v in obj["vars"]:
                o = v.get("origin")
                origin = None if o is None else (int(o["parent"]), int(o["factor"]), str(o["part"]))
                g.vars[int(v["id"])] = GVar(int(v["id"]), str(v["name"]), int(v["size"]), origin)
            for n in obj["nodes"]:
                kind = str(n["kind"])
                node = GNode(
                    id=int(n["id"]), kind=kind, name=str(n["name"]),
                    inputs=tuple(int(i) for i in n["inputs"]),
                    dims=tuple(int(d) for d in n["dims"]),
                    order=tuple(int(d) for d in n.get("order", ())),
                    staged=tuple(int(d) for d in n.get("staged", ())),
                )
                if kind in ("read", "write"):
                    node.slot = int(n["slot"])
                elif kind == "arith":
                    node.op = str(n["op"])
                    node.pre = str(n.get("pre", "identity"))
                    node.post = str(n.get("post", "identity"))
                    node.alpha = float(n.get("alpha", 0.0))
                    node.beta = float(n.get("beta", 1.0))
                elif kind == "view":
                    node.guarded = bool(n.get("guarded", False))
                    node.oob = float(n.get("oob", 0.0))
                    node.constraints = tuple(
                        GConstraint(int(c["input_dim"]),
                                    tuple((int(t[0]), int(t[1])) for t in c["terms"]),
                                    int(c.get("offset", 0)))
                        for c in n["constraints"])
                else:
                    raise GraphError(f"unknown node kind {kind!r}")
                g.nodes[node.id] = node
        except (KeyError, TypeError, ValueError, IndexError) as e:
            raise GraphError(f"malformed graph JSON: {e}") from None
        g._check()
        return g

    @classmethod
    def from_dfg(cls, dfg) -> "Graph":
        """Mirror a live ``loopsmith.ir.DFG`` by attribute reads only (no
        loopsmith import): node kinds are recognised by class name, exactly
        as serialize.py:54 spells them."""
        g = cls()
        ids: dict[int, int] = {}

        def vid(v) -> int:
            got = ids.get(v.uid)
            if got is not None:
                return got
            parent = None
            if v.origin is not None:
                parent = vid(v.origin.parent)
            i = len(ids)
            ids[v.uid] = i
            origin = None if v.origin is None else (parent, int(v.origin.factor), str(v.origin.part))
            g.vars[i] = GVar(i, str(v.name), int(v.size), origin)
            return i

        for nid in sorted(dfg.nodes):
            n = dfg.nodes[nid]
            k = n.kind
            kind = type(k).__name__.lower()
            node = GNode(id=int(n.id), kind=kind, name=str(n.output.name),
                         inputs=tuple(int(i) for i in n.inputs),
                         dims=tuple(vid(d) for d in n.output.dims),
                         order=tuple(vid(v) for v in n.order),
                         staged=tuple(sorted(vid(v) for v in n.staged)))
            if kind in ("read", "write"):
                node.slot = int(k.slot)
            elif kind == "arith":
                node.op, node.pre, node.post = str(k.op), str(k.pre), str(k.post)
                node.alpha, node.beta = float(k.alpha), float(k.beta)
            elif kind == "view":
                node.guarded, node.oob = bool(k.guarded), float(k.oob)
                node.constraints = tuple(
                    GConstraint(vid(c.input_dim), tuple((vid(v), int(co)) for v, co in c.terms),
                                int(c.offset))
                    for c in k.constraints)
            else:
                raise GraphError(f"unknown node kind {kind!r}")
            g.nodes[node.id] = node
        g._check()
        return g

    @classmethod
    def coerce(cls, obj) -> "Graph":
        """Graph | loopsmith DFG | LoopTree | JSON dict/str -> Graph."""
        if isinstance(obj, Graph):
            return obj
        if isinstance(obj, (dict, str, bytes)):
            return cls.from_json(obj)
        if hasattr(obj, "dfg") and hasattr(obj, "roots"):
            return cls.from_dfg(obj.dfg)
        if hasattr(obj, "nodes") and hasattr(obj, "splits"):
            return cls.from_dfg(obj)
        raise GraphError(f"cannot build a graph from {type(obj).__name__}")

    def _check(self) -> None:
        for n in self.nodes.values():
            for d in n.dims:
                if d not in self.vars:
                    raise GraphError(f"node {n.id}: unknown var {d}")
            for i in n.inputs:
                if i not in self.nodes:
                    raise GraphError(f"node {n.id}: unknown input {i}")
            if n.kind == "arith":
                if n.op not in OP_SEMANTICS:
                    raise GraphError(f"node {n.id}: unknown op {n.op!r}")
                for e in (n.pre, n.post):
                    if e not in ELEMENTWISE_OPS:
                        raise GraphError(f"node {n.id}: unknown elementwise op {e!r}")
        self.topo_order()

    # ---- queries ----------------------------------------------------------

    def __getitem__(self, nid: int) -> GNode:
        return self.nodes[nid]

    def size(self, vid: int) -> int:
        return self.vars[vid].size

    def shape(self, nid: int) -> tuple[int, ...]:
        return tuple(self.vars[d].size for d in self.nodes[nid].dims)

    def consumers(self, nid: int) -> list[GNode]:
        return [n for n in self.nodes.values() if nid in n.inputs]

    def reduction_dims(self, node: GNode) -> list[int]:
        """ir.py:321-332: dims on an input but not on the output (Arith only)."""
        if node.kind != "arith":
            return []
        out = set(node.dims)
        red: list[int] = []
        for i in node.inputs:
            for d in self.nodes[i].dims:
                if d not in out and d not in red:
                    red.append(d)
        return red

    def iteration_dims(self, node: GNode) -> list[int]:
        return list(node.dims) + self.reduction_dims(node)

    def topo_order(self) -> list[int]:
        """ir.py:349-369: Kahn's algorithm, ready set a min-heap on node id."""
        indeg = {nid: len(n.inputs) for nid, n in self.nodes.items()}
        cons: dict[int, list[int]] = {nid: [] for nid in self.nodes}
        for nid, n in self.nodes.items():
            for i in n.inputs:
                cons[i].append(nid)
        ready = [nid for nid, d in indeg.items() if d == 0]
        heapq.heapify(ready)
        out: list[int] = []
        while ready:
            nid = heapq.heappop(ready)
            out.append(nid)
            for c in cons[nid]:
                indeg[c] -= 1
                if indeg[c] == 0:
                    heapq.heappush(ready, c)
        if len(out) != len(self.nodes):
            raise GraphError("dataflow graph has a cycle")
        return out

    def slot_shapes(self) -> dict[int, tuple[int, ...]]:
        """feedback.py:46-52."""
        out: dict[int, tuple[int, ...]] = {}
        for n in self.nodes.values():
            if n.kind in ("read", "write"):
                out[n.slot] = self.shape(n.id)
        return out

    def input_slots(self) -> set[int]:
        return {n.slot for n in self.nodes.values() if n.kind == "read"}

    def output_slots(self) -> set[int]:
        return {n.slot for n in self.nodes.values() if n.kind == "write"}

    def write_of(self, nid: int) -> Optional[GNode]:
        for c in self.consumers(nid):
            if c.kind == "write":
                return c
        return None

    # ---- schedule lineage (tile hints only; results are schedule-free) ----

    def split_children(self, vid: int) -> Optional[tuple[int, int]]:
        outer = inner = None
        for v in self.vars.values():
            if v.origin is not None and v.origin[0] == vid:
                if v.origin[2] == "outer":
                    outer = v.id
                else:
                    inner = v.id
        if outer is None or inner is None:
            return None
        return outer, inner

    def inner_split_factor(self, vid: int) -> Optional[int]:
        """Innermost split factor applied to base var ``vid`` (None if never
        split): the reference's register-block width along that dim."""
        kids = self.split_children(vid)
        if kids is None:
            return None
        deeper = self.inner_split_factor(kids[1])
        return deeper if deeper is not None else self.vars[kids[1]].size

    # ---- analytics (feedback.py:177-227) ------------------------------------

    def count_flops(self) -> int:
        """feedback.py:177-214, restated on the mirror."""
        total = 0
        for node in self.nodes.values():
            if node.kind != "arith":
                continue
            red = self.reduction_dims(node)
            points = 1
            for d in list(node.dims) + red:
                points *= self.size(d)
            out_points = 1
            for d in node.dims:
                out_points *= self.size(d)
            combines = len(node.inputs) - 1
            accumulates = 1 if (red or node.alpha != 0.0) else 0
            if combines >= 1 and accumulates == 0:
                deferred = any(c.kind == "arith" and self.reduction_dims(c)
                               for c in self.consumers(node.id))
                if not deferred:
                    accumulates = 1
            per_point = combines + accumulates
            if node.beta != 1.0:
                per_point += 1
            total += points * per_point
            if node.post != "identity":
                total += out_points
            if node.alpha != 0.0 and node.pre != "identity":
                total += out_points
            if node.alpha not in (0.0, 1.0):
                total += out_points
        return total

    def bytes_moved(self) -> int:
        """feedback.py:217-227: 4 bytes per external element."""
        elems = 0
        for n in self.nodes.values():
            if n.kind in ("read", "write"):
                e = 1
                for s in self.shape(n.id):
                    e *= s
                elems += e
        return 4 * elems
