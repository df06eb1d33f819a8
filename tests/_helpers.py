"""Shared fixtures: reference-built indexes (oracle/_ref) on bf16-rounded KV and
their device mirrors.  The reference sees exactly the values the device
stores (bf16 rounded, widened to fp32), so selections, grafts and index
bytes must match bit for bit and only attention accumulation differs."""
from __future__ import annotations

import numpy as np

from oracle import refpy as R
from paper_2603_08453_b200 import api


def rounded_workload(n, d=128, seed=1, n_blobs=8, query_count=4, **kw):
    w = R.gen_workload(n, d, seed=seed, n_blobs=n_blobs, query_count=query_count, **kw)
    w.keys = api.bf16_round(w.keys)
    w.values = api.bf16_round(w.values)
    return w


def ref_engine(w, seed, **kw):
    return R.RefEngine(w.keys, w.values, w.text_code, seed=seed, **kw)


def host_index(ref: R.RefEngine) -> api.HostIndex:
    return api.HostIndex.from_export(ref.export())


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def assert_same_selection(got: api.RetrievalResult, ref: dict, ctx=""):
    assert got.degenerate == ref["degenerate"], ctx
    assert np.array_equal(got.selected_units, ref["units"]), (ctx, got.selected_units, ref["units"])
    assert np.array_equal(got.selected_clusters, ref["clusters"]), (
        ctx, got.selected_clusters[:20], ref["clusters"][:20])
    assert got.scanned_centroids == ref["scanned"], (ctx, got.scanned_centroids, ref["scanned"])
    if got.active_token_ids is not None:
        assert np.array_equal(got.active_token_ids, ref["active"]), (
            ctx, len(got.active_token_ids), len(ref["active"]))


def assert_same_index(a: api.HostIndex, e: R.IndexExport):
    assert np.array_equal(a.chunk_span, e.chunk_span)
    assert np.array_equal(a.cluster_of_chunk, e.cluster_of_chunk)
    assert np.array_equal(a.fine_centroid.view(np.uint32), e.fine_centroid.view(np.uint32))
    assert np.array_equal(a.fine_radius.view(np.uint64), e.fine_radius.view(np.uint64))
    assert np.array_equal(a.fine_token_count, e.fine_token_count)
    assert np.array_equal(a.fine_parent, e.fine_parent)
    assert np.array_equal(a.fine_member_off, e.fine_member_off)
    assert np.array_equal(a.fine_members, e.fine_members)
    assert np.array_equal(a.coarse_centroid.view(np.uint32), e.coarse_centroid.view(np.uint32))
    assert np.array_equal(a.coarse_radius.view(np.uint64), e.coarse_radius.view(np.uint64))
    assert np.array_equal(a.coarse_member_off, e.coarse_member_off)
    assert np.array_equal(a.coarse_members, e.coarse_members)
    assert np.array_equal(a.chunk_rep.view(np.uint32), e.chunk_rep.view(np.uint32))
