"""TKIX codec against the reference's serializer.

CPU: the host codec of liblychee_b200.so (lc_tkix_encode / lc_tkix_decode)
must produce exactly the reference's index_to_bytes (serialize.cpp:88-125)
for a reference-built index, before and after grafts, and decode it back
field for field.  GPU: a slot's live index (device build, uploads, grafts)
serialized on the device side equals the reference's bytes, and TKIX files
cross between the reference's save_index/load_index and lc_index_save/load.
"""
import os

import numpy as np
import pytest

from oracle import refpy as R
from paper_2603_08453_b200 import api

from ._helpers import assert_same_index, host_index, ref_engine, rounded_workload

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _cfg(seed, **kw):
    return api.IndexConfig(seed=seed, **kw)


@needs_ref
@pytest.mark.parametrize("n,d,seed", [(3000, 32, 5), (4096, 128, 21), (700, 16, 9)])
def test_encode_equals_reference_index_to_bytes(n, d, seed):
    w = R.gen_workload(n, d, seed=seed, n_blobs=4, query_count=2)
    ref = ref_engine(w, seed=seed)
    ours = api.index_to_bytes(host_index(ref), _cfg(seed))
    assert ours == ref.index_bytes()


@needs_ref
def test_encode_after_grafts_and_config_fields():
    w = R.gen_workload(2500, 64, seed=3, n_blobs=3, query_count=2)
    ref = R.RefEngine(w.keys, w.values, w.text_code, seed=3, max_units=9, iters=4, pooling=1)
    rng = np.random.default_rng(0)
    for i in range(70):  # 4 grafts of forced 16-token chunks
        k = rng.standard_normal(64).astype(np.float32)
        ref.push_and_graft(k / np.linalg.norm(k), rng.standard_normal(64).astype(np.float32))
    cfg = _cfg(3, max_coarse_units=9, kmeans_iters=4, pooling=1)
    assert api.index_to_bytes(host_index(ref), cfg) == ref.index_bytes()


@needs_ref
def test_decode_round_trip():
    w = R.gen_workload(3000, 32, seed=8, n_blobs=4, query_count=2)
    ref = ref_engine(w, seed=8)
    ix, cfg = api.index_from_bytes(ref.index_bytes())
    assert cfg == _cfg(8)
    assert_same_index(ix, ref.export())
    assert api.index_to_bytes(ix, cfg) == ref.index_bytes()


def test_decode_rejects_bad_input():
    with pytest.raises(api.L.LcError, match="not an index file"):
        api.index_from_bytes(b"XXXX" + b"\0" * 64)
    good = bytearray(b"TKIX")  # magic 0x58494b54, little-endian
    good += (1).to_bytes(4, "little") + (4).to_bytes(8, "little") + (3).to_bytes(8, "little")
    with pytest.raises(api.L.LcError, match="truncated"):
        api.index_from_bytes(bytes(good))


# ---------------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
@needs_ref
def test_device_slot_bytes_and_files(tmp_path):
    """Upload a reference index, graft on the device, and compare the slot's
    index_to_bytes with the reference after the same grafts; then move the
    state through TKIX files in both directions."""
    torch = pytest.importorskip("torch")
    w = rounded_workload(3000, 128, seed=4, n_blobs=3, query_count=2)
    ref = R.RefEngine(w.keys, w.values, w.text_code, seed=4)
    texts = ["\n" if c == 1 else ("}" if c == 2 else "") for c in w.text_code]
    st = api.StreamState(host_index(ref), w.keys, w.values, texts)
    st.engine.set_config(0, _cfg(4))
    assert st.engine.index_bytes(0) == ref.index_bytes()
    rng = np.random.default_rng(1)
    n0 = w.keys.shape[0]
    for i in range(80):
        k = api.bf16_round(rng.standard_normal(128).astype(np.float32))
        k = api.bf16_round(k / np.linalg.norm(k))
        v = api.bf16_round(rng.standard_normal(128).astype(np.float32))
        code = 1 if i % 11 == 5 else 0
        ref.push_and_graft(k, v, code)
        st.push_token(n0 + i, "\n" if code else "", k, v)
    assert st.graft_count >= 4
    assert st.engine.index_bytes(0) == ref.index_bytes()
    # device -> file -> reference load_index
    p1 = str(tmp_path / "dev.tkix")
    st.engine.save_index(0, p1, st.texts)
    back = R.RefEngine.load(p1)
    assert back.index_bytes() == ref.index_bytes()
    kb, vb = back.store()
    kr, vr = ref.store()
    assert np.array_equal(kb.view(np.uint32), kr.view(np.uint32))
    assert np.array_equal(vb.view(np.uint32), vr.view(np.uint32))
    # reference save_index -> lc_index_load into a fresh engine -> same retrieval
    p2 = str(tmp_path / "ref.tkix")
    ref.save(p2)
    n = ref.dims()[4]
    eng = api.Engine(1, 128, 2, cap_tokens=n + 8, cap_chunks=ref.dims()[1] + 8, cap_clusters=ref.dims()[2],
                     cap_units=64)
    got_texts = eng.load_index(0, p2)
    assert got_texts[:len(texts)] == texts
    assert eng.get_config(0) == _cfg(4)
    assert eng.index_bytes(0) == ref.index_bytes()
    q = torch.from_numpy(np.ascontiguousarray(w.queries[None, :2])).cuda()
    out = torch.zeros_like(q)
    b = api.Budgets(token_budget=256)
    eng.retrieve(q, b, out=out)
    for g in range(2):
        r = ref.retrieve(w.queries[g], token_budget=256)
        sel = eng.selection(0, g)
        assert np.array_equal(sel.selected_clusters, r["clusters"])
        assert np.array_equal(sel.active_token_ids, r["active"])
    os.remove(p1)
    os.remove(p2)
