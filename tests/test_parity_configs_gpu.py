"""Parity at the BASELINE.json configurations, on the GPU, against the reference.

* config 1 (32K, 8 KV heads x GQA 4, B = 2048): the committed fingerprints of
  SURVEY.md s8(d) (reference outputs for seeds 1000..1007) reproduced by the
  CUDA path in the reference-exact fp32 mode, and every head of every slot
  equal to the reference's retrieve() -- in fp32 mode and on the bench's own
  input path (GPU-generated bf16 workload + GPU build_index).
* config-2 shape (128K per slot: P = 64, ~800-2300 fine candidates per head):
  GPU-generated, GPU-built slots moved to the reference through a TKIX file
  (lc_index_save -> the reference's load_index), then every head's selection
  (units, clusters in rank order, scanned count, active ids) compared.
* 1M tokens per slot (config 4's context): the same, once with k_pickq's
  shared-memory key cap raised as the launch allows and once forced low, so
  both the on-chip and the L2 key paths of the largest heads are compared.
"""
import json
import os

import numpy as np
import pytest

from oracle import refpy as R
from paper_2603_08453_b200 import api

from . import golden_io
from ._helpers import assert_same_selection, host_index, ref_engine, rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
TOL = 1e-3


def texts_of(codes):
    return ["\n" if c == 1 else ("}" if c == 2 else "") for c in codes]


def _rows():
    return json.load(open(os.path.join(golden_io.HERE, "config1_fingerprints.json")))


def test_config1_fingerprints_fp32_mode():
    """8 slots x GQA 4 at 32K, the reference's own fp32 keys and index: query 0
    of each slot reproduces the committed fingerprint; all 4 heads equal the
    reference's retrieve()."""
    rows = _rows()
    S, G, n = len(rows), 4, 32768
    b = api.Budgets(token_budget=2048)
    ws = [R.gen_workload(n, 128, seed=r["seed"], query_count=G) for r in rows]
    refs = [ref_engine(w, seed=r["seed"]) for w, r in zip(ws, rows)]
    eng = api.Engine(S, 128, G, cap_tokens=n + 64, cap_chunks=n // 8 + 64, cap_clusters=n // 16 + 64,
                     cap_units=64, kv_f32=True)
    for s in range(S):
        assert format(R.fnv1a64(ws[s].keys.tobytes()), "016x") == rows[s]["keys_fnv1a"]
        assert refs[s].dims()[1:4] == [rows[s]["M"], rows[s]["L"], rows[s]["P"]]
        eng.upload_slot(s, host_index(refs[s]), ws[s].keys, ws[s].values)
    q = torch.from_numpy(np.stack([w.queries for w in ws])).cuda()
    out = torch.zeros_like(q)
    eng.retrieve(q, b, out=out)
    o = out.cpu().numpy()
    for s, row in enumerate(rows):
        for g, fp in enumerate(row["heads"]):
            got = eng.selection(s, g)
            assert got.selected_units.tolist() == fp["units"], (s, g)
            assert got.selected_clusters.tolist() == fp["clusters"], (s, g)
            assert len(got.active_token_ids) == fp["active"] and got.scanned_centroids == fp["scanned"], (s, g)
            assert np.allclose(o[s, g, :3], fp["out3"], rtol=0, atol=1e-6), (s, g)
            r = refs[s].retrieve(ws[s].queries[g], token_budget=2048)
            assert_same_selection(got, r, (s, g))
            assert rel_l2(o[s, g], r["output"]) < 1e-6
    assert eng.device_error() == 0


def _gpu_slots(n, seeds, G=4, keep_reps=True):
    """The bench's input path: GPU workload generator + GPU build_index."""
    S = len(seeds)
    cap_chunks = n // 8 + 64
    eng = api.Engine(S, 128, G, cap_tokens=n + 64, cap_chunks=cap_chunks, cap_clusters=(cap_chunks + 1) // 2,
                     cap_units=64, keep_reps=keep_reps)
    codes, qs = eng.gen_workload(n, np.array(seeds, np.uint64), query_count=G)
    spans = [api.segment_codes(codes[s]) for s in range(S)]
    eng.build_index([n] * S, spans, seeds)
    return eng, codes, qs


def _to_reference(eng, s, codes, tmp_path):
    p = str(tmp_path / f"slot{s}.tkix")
    eng.save_index(s, p, texts_of(codes[s]))
    ref = R.RefEngine.load(p)
    os.remove(p)
    return ref


def _compare_all(eng, refs, qs, b, out, slots):
    o = out.cpu().numpy()
    stats = []
    for s in slots:
        for g in range(eng.group):
            r = refs[s].retrieve(qs[s, g], token_budget=b.token_budget, unit_topk=b.unit_topk,
                                 sink=b.sink_size)
            got = eng.selection(s, g)
            assert_same_selection(got, r, (s, g))
            assert rel_l2(o[s, g], r["output"]) < TOL, (s, g)
            stats.append(r["scanned"])
    return stats


def test_config1_bench_path_bf16(tmp_path):
    """Config 1 through the bench's own path (bf16 K/V, GPU build)."""
    seeds = list(range(1000, 1008))
    eng, codes, qs = _gpu_slots(32768, seeds)
    refs = {s: _to_reference(eng, s, codes, tmp_path) for s in range(len(seeds))}
    q = torch.from_numpy(qs).cuda()
    out = torch.zeros_like(q)
    b = api.Budgets(token_budget=2048)
    eng.retrieve(q, b, out=out)
    _compare_all(eng, refs, qs, b, out, range(len(seeds)))
    assert eng.device_error() == 0


def test_config2_shape_128k(tmp_path):
    """Four 128K slots (config 2's per-slot shape: P = 64, hundreds to
    thousands of fine candidates per head), all 16 heads vs the reference."""
    seeds = [1000, 1077, 1150, 1255]
    n = 131072
    eng, codes, qs = _gpu_slots(n, seeds)
    refs = {s: _to_reference(eng, s, codes, tmp_path) for s in range(len(seeds))}
    assert all(refs[s].dims()[3] == 64 for s in refs)
    q = torch.from_numpy(qs).cuda()
    out = torch.zeros_like(q)
    for budget in (2048, 512):
        b = api.Budgets(token_budget=budget)
        eng.retrieve(q, b, out=out)
        scanned = _compare_all(eng, refs, qs, b, out, range(len(seeds)))
        assert max(scanned) - 64 > 500  # the fine tier is at config-2 scale
    assert eng.device_error() == 0


@pytest.fixture(scope="module")
def long_ctx(tmp_path_factory):
    n = 1 << 20
    seeds = [4242, 4243]
    eng, codes, qs = _gpu_slots(n, seeds)
    tmp = tmp_path_factory.mktemp("tkix1m")
    refs = {s: _to_reference(eng, s, codes, tmp) for s in range(len(seeds))}
    return eng, refs, qs


@pytest.mark.parametrize("keys_cap", [None, 512])
def test_long_context_1m(long_ctx, monkeypatch, keys_cap):
    """1M tokens per slot: thousands of fine candidates per head, through
    k_pickq's on-chip key path (cap raised as the launch allows) and its L2
    key path (cap forced low), vs the reference on the same index."""
    eng, refs, qs = long_ctx
    if keys_cap is not None:
        monkeypatch.setenv("LC_PICK_KEYS_CAP", str(keys_cap))
    q = torch.from_numpy(qs).cuda()
    out = torch.zeros_like(q)
    b = api.Budgets(token_budget=2048)
    eng.retrieve(q, b, out=out)
    scanned = _compare_all(eng, refs, qs, b, out, range(len(refs)))
    assert max(scanned) > 3000
    assert eng.device_error() == 0
