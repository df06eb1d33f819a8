"""CPU checks of bench.py's host logic: the configuration presets (BASELINE.json
configs 1, 2, 4, 5), the config-3 flush plan the streaming bench hands to the
device, and the layer-ordered slot layout the per-layer gather relies on."""
import argparse

import bench
from paper_2603_08453_b200 import api, shard


def _args(**kw):
    ns = dict(config=2, shards=0, tokens=None, layers=None, kv_heads=None, group=None, budget=None)
    ns.update(kw)
    return bench.apply_config(argparse.Namespace(**ns))


def test_config_presets():
    a = _args()
    assert (a.layers, a.kv_heads, a.group, a.tokens, a.budget) == (32, 8, 4, 131072, 2048)
    a = _args(config=1)
    assert (a.layers, a.tokens) == (1, 32768)
    a = _args(config=4)
    assert (a.layers, a.kv_heads, a.tokens, a.shards) == (36, 8, 1 << 20, 2)
    a = _args(config=5)
    assert a.shards == 8 and a.layers == 1
    # explicit flags win over the preset
    a = _args(config=4, tokens=65536, shards=4)
    assert (a.tokens, a.shards) == (65536, 4)
    assert bench.metric_of(_args()) == bench.METRIC
    assert "config4" in bench.metric_of(_args(config=4))


def test_stream_plan_follows_push_token():
    """streamer.cpp:29-66: buffer until max_len (16), then graft the head span
    of segment(buffer); a newline marker every 12 decoded tokens."""
    plan = bench.stream_takes(4101)
    assert len(plan) == 341
    buf = []
    it = iter(plan)
    nxt = next(it)
    for i in range(4101):
        buf.append("\n" if (i + 1) % 12 == 0 else "")
        if len(buf) >= 16:
            t, kd, lv = api.flush_take(buf)
            assert nxt == (i, t, kd, lv)
            buf = buf[t:]
            nxt = next(it, None)
    assert nxt is None
    assert all(8 <= t <= 16 for _, t, _, _ in plan)


def test_shard_of_config4_on_one_gpu():
    # config 4 on one GPU runs shard 0 of 2: half the KV heads of every layer
    slots = shard.slots_of_rank(0, 2, 36, 8, 1, order="layer")
    assert len(slots) == 144
    assert {s % 8 for s in slots} == {0, 1, 2, 3}
