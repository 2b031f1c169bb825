"""Row sharding of a contraction across ranks.

Output rows of a contraction are independent: rank r of P owns rows
[r0, r1) of A and C, B is replicated, and no data moves between ranks while
computing.  The only collective is the optional all-gather of the C shards
(NCCL over NVLink on the GPU box, gloo in the CPU tests), issued through
torch.distributed -- plumbing, not the hot path.
"""

from __future__ import annotations

import copy
import json


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of ``m`` rows: the first ``m % world`` ranks
    get one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of {world}")
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def shard_graph(graph, rows: int, var_name: str = "m") -> dict:
    """The same graph (reference JSON form) with base var ``var_name`` resized
    to ``rows``; split children are resized consistently (schedule.py:23-43:
    inner = factor, outer = ceil(size / factor))."""
    obj = json.loads(graph) if isinstance(graph, (str, bytes)) else copy.deepcopy(graph)
    base = [v for v in obj["vars"] if v["name"] == var_name and v["origin"] is None]
    if len(base) != 1:
        raise ValueError(f"graph has no unique base var {var_name!r}")
    sizes = {base[0]["id"]: rows}
    changed = True
    while changed:
        changed = False
        for v in obj["vars"]:
            o = v["origin"]
            if o is not None and o["parent"] in sizes and v["id"] not in sizes:
                psize = sizes[o["parent"]]
                v["size"] = o["factor"] if o["part"] == "inner" else -(-psize // o["factor"])
                sizes[v["id"]] = v["size"]
                changed = True
    base[0]["size"] = rows
    return obj


def gather_rows(local, world: int, group=None):
    """All-gather equal-row C shards (torch tensors) into the full matrix on
    every rank.  Uneven shards are padded to the largest shard."""
    import torch
    import torch.distributed as dist
    rows = torch.tensor([local.shape[0]], device=local.device)
    sizes = [torch.zeros_like(rows) for _ in range(world)]
    dist.all_gather(sizes, rows, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    if local.shape[0] < mx:
        pad = torch.zeros((mx - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        local = torch.cat([local, pad])
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        parts = list(out.split(mx))
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def nccl_comm(group=None):
    """The library's own NCCL communicator over the ranks of a torch.distributed
    group (rank 0 makes the unique id, broadcast as an object): the handle
    lsb_allgather_rows gathers C row shards with."""
    import torch.distributed as dist
    from . import native
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [native.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return native.NcclComm(rank, world, box[0])


def gather_rows_native(comm, local, out, stream: int = 0) -> None:
    """All-gather equal row shards (contiguous torch CUDA tensors, ``out`` of
    comm.nranks x local's rows) through lsb_allgather_rows."""
    if not (local.is_contiguous() and out.is_contiguous()) or out.numel() != local.numel() * comm.nranks:
        raise ValueError("gather_rows_native needs contiguous equal shards and a nranks-times output")
    comm.allgather_rows(local.data_ptr(), out.data_ptr(), local.numel(), stream)
