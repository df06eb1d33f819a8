"""Multi-GPU partitioning of the decode-step path.

Every (layer, KV head, sequence) slot is independent, so the path shards with
no per-step collective: rank r owns KV heads {h : h*R // H_kv == r} of every
layer and sequence.  The only exchange is the all-gather of head outputs at
the layer boundary (torch.distributed: NCCL on GPUs, gloo in tests), done
per layer by LayerGather, or once per step for a step that runs every layer's
slots in one launch (gather_outputs).
"""
from __future__ import annotations


def slot_id(seq: int, layer: int, head: int, layers: int, kv_heads: int) -> int:
    """Global slot id of (sequence, layer, KV head)."""
    return (seq * layers + layer) * kv_heads + head


def slots_of_rank(rank: int, world: int, layers: int, kv_heads: int, batch: int = 1, order: str = "seq"):
    """Global slot ids owned by `rank`.

    order "seq": ascending slot id, i.e. (sequence, layer, head) order.
    order "layer": (layer, sequence, head) order, so one layer's local slots
    are contiguous -- the layout a layer-by-layer decode launches and gathers.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    heads = [h for h in range(kv_heads) if (h * world) // kv_heads == rank]
    if order == "seq":
        return [slot_id(b, l, h, layers, kv_heads) for b in range(batch) for l in range(layers) for h in heads]
    if order == "layer":
        return [slot_id(b, l, h, layers, kv_heads) for l in range(layers) for b in range(batch) for h in heads]
    raise ValueError("order must be 'seq' or 'layer'")


def gather_outputs(local_out, rank: int, world: int, layers: int, kv_heads: int, batch: int = 1):
    """All-gather every rank's [n_local, G, d] outputs (order "seq") and scatter
    them back into global slot order -> [n_slots, G, d] on every rank."""
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


class LayerGather:
    """The layer-boundary exchange of a layer-by-layer decode: after layer l's
    slots are attended, one all_gather_into_tensor collects every rank's
    contiguous rows of that layer (local order "layer") into a preallocated
    [layers][world * rows_per_layer][...] buffer.  The collective reads and
    writes fixed buffers, so a whole step of them is CUDA-graph capturable
    under NCCL.  `layer_view(l)` returns layer l's gathered rows in global
    (sequence, head) order, the order the next layer's projection consumes."""

    def __init__(self, rank, world, layers, kv_heads, batch, row_shape, dtype, device, group=None):
        import torch

        if kv_heads % world:
            raise ValueError("the world size must divide the KV heads")
        self.rank, self.world, self.layers, self.kv_heads, self.batch = rank, world, layers, kv_heads, batch
        self.hpr = kv_heads // world
        self.rows = batch * self.hpr  # local rows of one layer
        self.group = group
        self.buf = torch.zeros((layers, world * self.rows) + tuple(row_shape), dtype=dtype, device=device)
        # gathered row (r, b, k) holds (sequence b, head r*hpr + k): position in (b, head) order
        perm = [0] * (world * self.rows)
        for r in range(world):
            for b in range(batch):
                for k in range(self.hpr):
                    perm[b * kv_heads + r * self.hpr + k] = (r * batch + b) * self.hpr + k
        self.perm = torch.tensor(perm, device=device)

    def local_rows(self, layer):
        """Slice of the engine's local slot rows that holds `layer` (order "layer")."""
        return slice(layer * self.rows, (layer + 1) * self.rows)

    def gather(self, out_local, layer):
        """out_local: the engine's [n_local, G, d] output; all-gathers layer's rows."""
        import torch.distributed as dist

        src = out_local[self.local_rows(layer)]
        if self.world == 1:
            self.buf[layer].copy_(src)
            return
        dist.all_gather_into_tensor(self.buf[layer], src, group=self.group)

    def layer_view(self, layer):
        """[batch * kv_heads, ...] of `layer` in global (sequence, head) order."""
        return self.buf[layer].index_select(0, self.perm)
