"""CPU oracle for the B200 backend -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The B200 backend (``paper_2205_00618_b200``) never calls into ``oracle/``.

It restates the reference's schedule-independent f64 interpreter,
``loopsmith.feedback.reference_eval`` (reference
``pkg/src/loopsmith/feedback.py:69-170``), on the neutral graph mirror
(``paper_2205_00618_b200.graph.Graph``), with two additions that keep the
semantics but bound memory so the BASELINE-sized configs can be checked:

  * ``restrict``: evaluate only selected coordinates of chosen iteration vars
    (row blocks / sampled rows and columns of the output);
  * reduction chunking: the reference materialises the whole iteration space
    (``[M,K,N]`` f64, 8 GiB at 1024^3); here the largest reduction dim is
    processed in chunks and the chunk results are folded with the same reduce
    op (exact for max/min, f64 re-association for add -- far below the fp32
    tolerance).  (mul, add) over two operands takes the f64 BLAS path
    (``np.einsum``), which SURVEY.md §8(c) accepts as a restatement.

Parity of this restatement is pinned against outputs of the real reference
(``reference_eval`` and the reference VM) stored under ``tests/golden/`` by
``tests/golden/make_golden.py``; see ``tests/test_oracle.py``.
"""

from __future__ import annotations

import os
import sys
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2205_00618_b200.graph import Graph, OP_IDENTITY  # noqa: E402  (parsing only)


class OracleError(Exception):
    pass


# feedback.py:25-43
_EW = {
    "identity": lambda x: x,
    "relu": lambda x: np.maximum(x, 0.0),
    "sigmoid": lambda x: 1.0 / (1.0 + np.exp(-x)),
}
_COMBINE = {"add": np.add, "mul": np.multiply, "max": np.maximum, "min": np.minimum}
_REDUCE = {"add": np.sum, "mul": np.prod, "max": np.max, "min": np.min}

#: elements of f64 scratch one chunk of a broadcast reduction may hold
CHUNK_ELEMS = 1 << 24


class _Val:
    """An evaluated node: f64 array whose axis i runs over ``sel[dims[i]]``."""

    __slots__ = ("arr", "dims")

    def __init__(self, arr: np.ndarray, dims: tuple[int, ...]):
        self.arr = arr
        self.dims = dims


def _sel(g: Graph, restrict: dict, vid: int) -> np.ndarray:
    s = restrict.get(vid)
    if s is None:
        return np.arange(g.size(vid))
    return np.asarray(s, dtype=np.int64)


def _align(arr: np.ndarray, have: tuple, want: list) -> np.ndarray:
    """feedback.py:111-118: transpose/expand ``arr`` into axis order ``want``."""
    have = list(have)
    perm = [have.index(d) for d in want if d in have]
    moved = np.transpose(arr, perm) if arr.ndim else arr
    present = [d for d in want if d in have]
    shape = [moved.shape[present.index(d)] if d in have else 1 for d in want]
    return moved.reshape(shape)


def reference_eval(g, buffers: dict, restrict: Optional[dict] = None) -> dict:
    """Restatement of feedback.py:69-108.

    ``g``: Graph or anything ``Graph.coerce`` accepts.  ``buffers``: slot ->
    array (inputs required; write slots optional, seeding ``c_in``).
    ``restrict``: var id -> sorted coordinate array; outputs are returned over
    the restricted coordinates only.  Returns slot -> f64 array.
    """
    g = Graph.coerce(g)
    restrict = dict(restrict or {})
    shapes = g.slot_shapes()
    for slot, shape in shapes.items():
        if slot in buffers and np.asarray(buffers[slot]).size != int(np.prod(shape)):
            raise OracleError(f"slot {slot}: expected {shape}")

    prior: dict[int, np.ndarray] = {}
    write_of: dict[int, int] = {}
    for node in g.nodes.values():
        if node.kind == "write":
            arr = buffers.get(node.slot)
            shape = shapes[node.slot]
            full = (np.zeros(shape) if arr is None
                    else np.asarray(arr, dtype=np.float64).reshape(shape))
            prior[node.slot] = _take(g, restrict, full, node.dims)
            write_of[node.inputs[0]] = node.id

    vals: dict[int, _Val] = {}
    outs: dict[int, np.ndarray] = {}
    for nid in g.topo_order():
        node = g[nid]
        if node.kind == "read":
            full = np.asarray(buffers[node.slot], dtype=np.float64).reshape(shapes[node.slot])
            vals[nid] = _Val(_take(g, restrict, full, node.dims), node.dims)
        elif node.kind == "view":
            vals[nid] = _eval_view(g, restrict, node, vals[node.inputs[0]])
        elif node.kind == "arith":
            vals[nid] = _eval_arith(g, restrict, node, vals, prior, write_of)
        elif node.kind == "write":
            src = vals[node.inputs[0]]
            outs[node.slot] = np.ascontiguousarray(_align(src.arr, src.dims, list(node.dims)))
    return outs


def _take(g: Graph, restrict: dict, arr: np.ndarray, dims) -> np.ndarray:
    for ax, d in enumerate(dims):
        if d in restrict:
            arr = np.take(arr, _sel(g, restrict, d), axis=ax)
    return arr


def _eval_view(g: Graph, restrict: dict, node, src: _Val) -> _Val:
    """feedback.py:121-141, over restricted output coordinates."""
    out_dims = list(node.dims)
    sels = [_sel(g, restrict, d) for d in out_dims]
    grids = np.meshgrid(*sels, indexing="ij") if sels else []
    pos = {d: grids[i] for i, d in enumerate(out_dims)}
    out_shape = tuple(len(s) for s in sels)
    in_range = np.ones(out_shape, dtype=bool)
    idxs = []
    src_dims = list(src.dims)
    for c in node.constraints:
        x = np.full(out_shape, c.offset, dtype=np.int64)
        for v, coeff in c.terms:
            x = x + coeff * pos[v]
        size = g.size(c.input_dim)
        in_range &= (x >= 0) & (x < size)
        x = np.clip(x, 0, size - 1)
        if c.input_dim in restrict:  # source axis holds only selected coords
            sel = _sel(g, restrict, c.input_dim)
            lut = np.full(size, -1, dtype=np.int64)
            lut[sel] = np.arange(len(sel))
            local = lut[x]
            if np.any((local < 0) & in_range):
                raise OracleError(f"view {node.id} needs coordinates outside the restriction")
            x = np.maximum(local, 0)
        idxs.append((src_dims.index(c.input_dim), x))
    idxs.sort(key=lambda t: t[0])
    got = src.arr[tuple(x for _, x in idxs)]
    if node.guarded:
        got = np.where(in_range, got, node.oob)
    elif not in_range.all():
        raise OracleError(f"view {node.id} accesses out of range")
    return _Val(np.asarray(got, dtype=np.float64), tuple(out_dims))


def _eval_arith(g: Graph, restrict: dict, node, vals, prior, write_of) -> _Val:
    """feedback.py:144-170 with reduction chunking (see module docstring)."""
    space = g.iteration_dims(node)
    out_n = len(node.dims)
    red = space[out_n:]
    parts = [vals[i] for i in node.inputs]
    comb, redop = node.combine_op, node.reduce_op

    if red:
        reduced = _reduce_chunked(g, restrict, node, parts, space, comb, redop)
    else:
        aligned = [_align(p.arr, p.dims, space) for p in parts]
        combined = aligned[0]
        for p in aligned[1:]:
            combined = _COMBINE[comb](combined, p)
        if node.beta != 1.0:
            combined = node.beta * combined
        reduced = np.broadcast_to(combined, tuple(len(_sel(g, restrict, d)) for d in space))
    if node.alpha != 0.0:
        wid = write_of.get(node.id)
        if wid is None:
            raise OracleError(f"node {node.id} has alpha != 0 but no write consumer")
        w = g[wid]
        c_in = _align(prior[w.slot], w.dims, list(node.dims))
        init = node.alpha * _EW[node.pre](c_in)
        reduced = _COMBINE[redop](init, reduced)
    return _Val(np.asarray(_EW[node.post](reduced), dtype=np.float64), tuple(node.dims))


def _reduce_chunked(g, restrict, node, parts, space, comb, redop) -> np.ndarray:
    out_n = len(node.dims)
    sizes = [len(_sel(g, restrict, d)) for d in space]
    red_axes = tuple(range(out_n, len(space)))
    # fast path: two-operand (mul, add) contraction through f64 BLAS
    carried = {d for p in parts for d in p.dims}
    if (comb == "mul" and redop == "add" and len(parts) == 2 and node.beta == 1.0
            and all(d in carried for d in node.dims)):
        letters = {d: chr(ord("a") + i) for i, d in enumerate(space)}
        spec = ",".join("".join(letters[d] for d in p.dims) for p in parts)
        outspec = "".join(letters[d] for d in node.dims)
        r = np.einsum(f"{spec}->{outspec}", parts[0].arr, parts[1].arr, optimize=True)
        return np.broadcast_to(r, tuple(sizes[:out_n]))

    total = int(np.prod(sizes)) if sizes else 1
    # chunk along the largest reduction axis
    ax = max(red_axes, key=lambda a: sizes[a])
    per = max(1, total // max(sizes[ax], 1))
    step = max(1, CHUNK_ELEMS // per)
    acc = None
    for lo in range(0, sizes[ax], step):
        hi = min(sizes[ax], lo + step)
        aligned = []
        for p in parts:
            a = _align(p.arr, p.dims, space)
            if a.shape[ax] != 1:
                a = a[(slice(None),) * ax + (slice(lo, hi),)]
            aligned.append(a)
        combined = aligned[0]
        for p in aligned[1:]:
            combined = _COMBINE[comb](combined, p)
        if node.beta != 1.0:
            combined = node.beta * combined
        shape = list(sizes)
        shape[ax] = hi - lo
        combined = np.broadcast_to(combined, tuple(shape))
        part = _REDUCE[redop](combined, axis=red_axes)
        acc = part if acc is None else _COMBINE[redop](acc, part)
    return acc


# --------------------------------------------------------------------------
# parity rules (BASELINE.json north_star)
# --------------------------------------------------------------------------

#: fp32 sum-reduction tolerance from north_star: 1e-4 relative / 1e-5 absolute
RTOL, ATOL = 1e-4, 1e-5


def strict_ok(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Per-element |d| <= 1e-5 + 1e-4*|ref| against the f64 oracle."""
    got = np.asarray(got, dtype=np.float64).reshape(ref.shape)
    same_inf = np.isinf(ref) & (got == ref)
    return same_inf | (np.abs(got - ref) <= ATOL + RTOL * np.abs(ref))


def ref_metric(got: np.ndarray, ref: np.ndarray) -> float:
    """test_acceptance.py:57-58: max |d| / max(|ref|, 1)."""
    got = np.asarray(got, dtype=np.float64).reshape(ref.shape)
    fin = np.isfinite(ref)
    if not fin.all():
        if not np.array_equal(got[~fin], ref[~fin]):
            return float("inf")
    if not fin.any():
        return 0.0
    return float(np.max(np.abs(got[fin] - ref[fin]) / np.maximum(np.abs(ref[fin]), 1.0)))


def bit_exact(got: np.ndarray, ref: np.ndarray) -> bool:
    """Max/min semirings: f32 result equals float32(f64 oracle) bit for bit."""
    want = np.asarray(ref, dtype=np.float64).astype(np.float32)
    got = np.asarray(got, dtype=np.float32).reshape(want.shape)
    return bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))
