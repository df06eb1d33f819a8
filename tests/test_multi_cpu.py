"""CPU: KV-head sharding and the layer-boundary all-gather over gloo, world size 2."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08453_b200 import shard


def test_slots_partition_all_heads():
    for world in (1, 2, 4, 8):
        owned = [shard.slots_of_rank(r, world, 32, 8) for r in range(world)]
        flat = sorted(s for o in owned for s in o)
        assert flat == list(range(256))
        assert all(len(o) == 256 // world for o in owned)
        # a rank owns whole KV heads across all layers
        for r, o in enumerate(owned):
            heads = {s % 8 for s in o}
            assert len(heads) == 8 // world


def test_weak_scaling_keeps_per_gpu_load():
    # bench.py's default at N GPUs: batch = N, so every rank keeps 256 slots
    # (one sequence's worth), whole KV heads of every sequence
    for world in (1, 2, 4, 8):
        owned = [shard.slots_of_rank(r, world, 32, 8, batch=world) for r in range(world)]
        assert all(len(o) == 256 for o in owned)
        flat = sorted(s for o in owned for s in o)
        assert flat == list(range(256 * world))
        for o in owned:
            seqs = {s // 256 for s in o}
            assert seqs == set(range(world))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layers, heads, G, d = 4, 8, 4, 16
    mine = shard.slots_of_rank(rank, world, layers, heads)
    local = torch.stack([torch.full((G, d), float(s)) for s in mine])
    full = shard.gather_outputs(local, rank, world, layers, heads)
    ok = all(bool((full[s] == float(s)).all()) for s in range(layers * heads))
    q.put((rank, ok, full.shape[0]))
    dist.destroy_process_group()


def test_allgather_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res) and all(r[2] == 32 for r in res)


def test_layer_order_contiguous():
    # order "layer": one layer's local slots are contiguous, every (seq, head) once
    for world in (1, 2, 4):
        for batch in (1, 3):
            mine = shard.slots_of_rank(0, world, 5, 8, batch, order="layer")
            assert sorted(mine) == shard.slots_of_rank(0, world, 5, 8, batch)
            rows = batch * 8 // world
            for l in range(5):
                blk = mine[l * rows:(l + 1) * rows]
                assert {(s // 8) % 5 for s in blk} == {l}


def _layer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layers, heads, batch, G, d = 3, 4, 2, 2, 8
    mine = shard.slots_of_rank(rank, world, layers, heads, batch, order="layer")
    # the engine's output rows in local slot order, tagged with the global slot id
    out = torch.stack([torch.full((G, d), float(s)) for s in mine])
    lg = shard.LayerGather(rank, world, layers, heads, batch, (G, d), torch.float32, "cpu")
    ok = True
    for l in range(layers):
        lg.gather(out, l)
        v = lg.layer_view(l)
        for b in range(batch):
            for h in range(heads):
                ok &= bool((v[b * heads + h] == float(shard.slot_id(b, l, h, layers, heads))).all())
    q.put((rank, ok))
    dist.destroy_process_group()


def test_layer_gather_world2_gloo():
    """bench.py's layer-boundary exchange (shard.LayerGather, one all-gather
    per layer over the local layer-ordered rows) reassembles every layer's
    head outputs in global (sequence, head) order on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_layer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res)
