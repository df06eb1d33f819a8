"""Multi-GPU partitioning of the decode-step path.

Every (layer, KV head, sequence) slot is independent, so the path shards with
no per-step collective: rank r owns KV heads {h : h*R // H_kv == r} of every
layer and sequence.  The only exchange is the all-gather of head outputs at
the layer boundary (torch.distributed, NCCL on GPUs / gloo in tests).
"""
from __future__ import annotations


def slots_of_rank(rank: int, world: int, layers: int, kv_heads: int, batch: int = 1):
    """Global slot ids (slot = (seq*layers + layer)*kv_heads + head) owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    n = layers * kv_heads * batch
    return [s for s in range(n) if ((s % kv_heads) * world) // kv_heads == rank]


def gather_outputs(local_out, rank: int, world: int, layers: int, kv_heads: int, batch: int = 1):
    """All-gather every rank's [n_local, G, d] outputs and scatter them back into
    global slot order -> [n_slots, G, d] on every rank."""
    import torch
    import torch.distributed as dist

    parts = [torch.empty_like(local_out) for _ in range(world)] if world > 1 else [local_out]
    if world > 1:
        # ranks own equal slot counts when world divides kv_heads
        dist.all_gather(parts, local_out.contiguous())
    n = layers * kv_heads * batch
    out = torch.empty((n,) + tuple(local_out.shape[1:]), dtype=local_out.dtype, device=local_out.device)
    for r in range(world):
        idx = torch.tensor(slots_of_rank(r, world, layers, kv_heads, batch), device=local_out.device)
        out[idx] = parts[r]
    return out
