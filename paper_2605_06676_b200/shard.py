"""Multi-GPU partitioning of the eviction path (host-side logic, no data-path collective).

Every (seq, layer, kv-head) is independent for scoring, top-k, compaction and decode; the one
global coupling, LKV-H's threshold over all L*H logits (policy.cpp:118), is recomputed
redundantly and bit-identically on every rank from the same logits.  Ranks therefore only
need to agree on *who owns which heads*:

* batch sharding (weak scaling, bench default): sequence s -> rank s % world;
* layer-range head sharding (one long sequence over N GPUs): contiguous layer
  ranges, uniform scoring work because t is uniform within a sequence;
* LPT over (seq, head) by retained rows for decode, where work is proportional to the
  budget (known before eviction).
"""
from __future__ import annotations


def batch_shard(n_seq: int, world: int, rank: int) -> list:
    """Sequences owned by `rank` (round-robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return [s for s in range(n_seq) if s % world == rank]


def layer_ranges(n_layers: int, world: int) -> list:
    """Contiguous [l0, l1) layer range per rank; sizes differ by at most one."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(n_layers, world)
    out, l0 = [], 0
    for r in range(world):
        l1 = l0 + base + (1 if r < extra else 0)
        out.append((l0, l1))
        l0 = l1
    return out


def lpt_assign(weights, world: int) -> list:
    """Deterministic longest-processing-time-first assignment: items by weight descending
    (ties -> lower index) each go to the currently least-loaded rank (ties -> lower rank).
    Returns the owning rank per item."""
    order = sorted(range(len(weights)), key=lambda i: (-weights[i], i))
    load = [0] * world
    owner = [0] * len(weights)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += weights[i]
    return owner


def imbalance(weights, owner, world: int) -> float:
    """max rank load / mean rank load (1.0 = perfect)."""
    load = [0] * world
    for w, r in zip(weights, owner):
        load[r] += w
    mean = sum(load) / world if world else 0
    return max(load) / mean if mean else 1.0


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over the default process group (the timing rule: slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
