"""GPU prefill helpers vs the reference: workload generator and build_index.

* lc_index_build must reproduce the reference's build_index bit for bit
  (every field index_to_bytes serializes, serialize.cpp:88-125) from the same
  keys: chunk reps, k-means (init, Lloyd rounds, empty repair), radii, tiers.
* lc_gen_workload must reproduce gen_clustered_workload's control stream
  (markers, queries) exactly and its K/V up to the documented last-bit
  differences of CUDA's fp64 log/sin/cos (measured: none at these sizes).
"""
import numpy as np
import pytest

from oracle import refpy as R
from paper_2603_08453_b200 import api

from ._helpers import assert_same_index, assert_same_selection, rel_l2, rounded_workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def texts_of(codes):
    return ["\n" if c == 1 else ("}" if c == 2 else "") for c in codes]


def test_gen_workload_matches_reference_generator():
    seeds = [5, 6, 1000]
    n = 4096
    eng = api.Engine(len(seeds), 128, 4, cap_tokens=n, cap_chunks=n // 4, cap_clusters=n // 8, cap_units=64)
    codes, qs = eng.gen_workload(n, seeds)
    total = bad_k = bad_v = 0
    for s, seed in enumerate(seeds):
        w = R.gen_workload(n, 128, seed=seed, query_count=4)
        assert np.array_equal(codes[s], w.text_code)
        assert np.array_equal(qs[s], w.queries)
        kb, vb = eng.kv_download(s, n)
        bad_k += int((kb != api.bf16_bits(w.keys)).sum())
        bad_v += int((vb != api.bf16_bits(w.values)).sum())
        total += kb.size
    assert bad_k <= total * 1e-6 and bad_v <= total * 1e-6, (bad_k, bad_v, total)


@pytest.mark.parametrize("iters", [10, 3])
def test_gpu_build_index_bit_exact(iters):
    cases = [(3000, 11), (5000, 12), (8192, 1000), (700, 13)]
    S = len(cases)
    nmax = max(n for n, _ in cases)
    eng = api.Engine(S, 128, 4, cap_tokens=nmax, cap_chunks=nmax // 4, cap_clusters=nmax // 8, cap_units=64)
    ws, spans = [], []
    for s, (n, seed) in enumerate(cases):
        w = rounded_workload(n, 128, seed=seed, query_count=4)
        eng.kv_upload(s, w.keys, w.values)
        spans.append(api.segment(texts_of(w.text_code)))
        ws.append(w)
    eng.build_index([n for n, _ in cases], spans, [seed for _, seed in cases], kmeans_iters=iters)
    b = api.Budgets(token_budget=512)
    q = torch.from_numpy(np.stack([w.queries for w in ws])).cuda()
    out = torch.zeros_like(q)
    eng.retrieve(q, b, out=out)
    o = out.cpu().numpy()
    for s, (n, seed) in enumerate(cases):
        ref = R.RefEngine(ws[s].keys, ws[s].values, ws[s].text_code, seed=seed, iters=iters)
        assert_same_index(eng.download_slot(s), ref.export())
        for g in range(4):
            r = ref.retrieve(ws[s].queries[g], token_budget=512)
            assert_same_selection(eng.selection(s, g), r, (s, g))
            assert rel_l2(o[s, g], r["output"]) < 1e-3


def test_gpu_generated_then_built_matches_reference_build():
    """End to end on the bench's input path: GPU workload + GPU build == the
    reference's build_index fed the very same (downloaded) keys."""
    seeds = [2024, 2025]
    n = 6000
    eng = api.Engine(len(seeds), 128, 4, cap_tokens=n, cap_chunks=n // 4, cap_clusters=n // 8, cap_units=64)
    codes, qs = eng.gen_workload(n, seeds)
    spans = [api.segment(texts_of(codes[s])) for s in range(len(seeds))]
    eng.build_index([n] * len(seeds), spans, seeds)
    for s, seed in enumerate(seeds):
        kb, vb = eng.kv_download(s, n)
        keys = (kb.astype(np.uint32) << 16).view(np.float32)
        vals = (vb.astype(np.uint32) << 16).view(np.float32)
        ref = R.RefEngine(keys, vals, codes[s], seed=seed)
        assert_same_index(eng.download_slot(s), ref.export())
