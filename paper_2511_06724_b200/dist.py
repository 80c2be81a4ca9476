"""Host-side multi-GPU plumbing around libargus (one process per GPU).

The data path (scan, merge, predictor, assignment, NCCL broadcast/all-gather)
lives in libargus.so; this module only holds the host protocol that callers and
bench.py share: the striped cache layout (global id g on rank g mod G at slot
g div G), distribution of the NCCL unique id over the caller's
process group, and max-over-ranks timing.  Tested with world_size=2 gloo on CPU
(tests/test_multi_gloo.py).
"""
from __future__ import annotations


def cache_position(g: int, capacity: int = 0, evict: bool = False) -> int:
    """Cache position of global id g: g itself, or g mod capacity for a ring-evicting
    cache (argus_config.evict; capacity % world == 0)."""
    return g % capacity if evict else g


def stripe_owner(g: int, world: int, capacity: int = 0, evict: bool = False) -> int:
    """Rank holding global cache id g."""
    return cache_position(g, capacity, evict) % world


def stripe_slot(g: int, world: int, capacity: int = 0, evict: bool = False) -> int:
    """Local row of global id g on its owner."""
    return cache_position(g, capacity, evict) // world


def live_ids(M: int, capacity: int, evict: bool) -> range:
    """Global ids held after M inserts: all of them, or the last `capacity` (ring)."""
    return range(max(0, M - capacity), M) if evict else range(M)


def local_rows(M: int, world: int, rank: int) -> int:
    """Rows of an M-entry cache held by `rank` (shards differ by at most one)."""
    return (M + world - 1 - rank) // world


def share_nccl_id(dist, rank: int, make_id):
    """Rank 0 creates the 128-byte ncclUniqueId, every rank returns the same bytes."""
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, value: float, device=None) -> float:
    """Max of a per-rank float (elapsed ms) over the group: the job's time."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
