"""Multi-GPU placement of the reuse prefill.

The reference has no parallelism; independent requests are
the unit that shards.  One process per GPU, each with a full weight replica and a
replicated device store; rank r serves requests r, r + world, ... in one batched
device pass (`prefill_batch_with_reuse`).  There is no collective on the data path:
the only cross-rank traffic is the timing barrier and the max-over-ranks reduction
of the benchmark, and an optional host-side gather of the results' metadata.
"""
from __future__ import annotations

import numpy as np


def shard_indices(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin shard of n_items independent requests onto `world` ranks."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, n_items, world))


def head_split(heads: int, world: int) -> list[tuple[int, int]]:
    """(first head, count) per rank for a head-parallel split; uneven when world does not
    divide heads (28 heads on 8 ranks -> 4,4,4,4,3,3,3,3)."""
    if world <= 0 or world > heads:
        raise ValueError(f"cannot split {heads} heads over {world} ranks")
    base, extra = divmod(heads, world)
    out, h0 = [], 0
    for r in range(world):
        k = base + (1 if r < extra else 0)
        out.append((h0, k))
        h0 += k
    return out


def run_shard(model, requests, store, rank: int, world: int):
    """This rank's results: prefill_batch_with_reuse over its shard (no collective)."""
    from .engine import prefill_batch_with_reuse
    idx = shard_indices(len(requests), rank, world)
    return idx, prefill_batch_with_reuse(model, [requests[i] for i in idx], store) if idx else []


def gather_metadata(idx, results, group=None):
    """Host-side gather of (request index, positions, computed_per_layer) to every rank,
    ordered by request index (torch.distributed object collective; any backend)."""
    import torch.distributed as dist
    mine = [(i, np.asarray(r.positions).tolist(), list(r.metrics.computed_per_layer))
            for i, r in zip(idx, results)]
    world = dist.get_world_size(group)
    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    return sorted((t for part in allv for t in part), key=lambda t: t[0])
