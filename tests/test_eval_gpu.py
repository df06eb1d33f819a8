"""GPU evaluator vs the reference's evaluator.cpp.

audit_ub_soundness counts and oracle_topk_tokens id sets must equal the
reference's exactly (sequential fp64 dots on both sides); full_attention is
within the attention tolerance (fp32 accumulation over bf16 K/V)."""
import numpy as np
import pytest

from oracle import refpy as R
from paper_2603_08453_b200 import api

from ._helpers import host_index, ref_engine, rel_l2, rounded_workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def case():
    w = rounded_workload(8192, 128, seed=31, n_blobs=6, query_count=4)
    ref = ref_engine(w, seed=31)
    eng = api.Engine(1, 128, 4, cap_tokens=8192 + 64, cap_chunks=2048, cap_clusters=1024, cap_units=64)
    eng.upload_slot(0, host_index(ref), w.keys, w.values)
    rng = np.random.default_rng(5)
    qs = rng.standard_normal((40, 128)).astype(np.float32)
    qs = np.concatenate([qs, w.queries])
    return w, ref, eng, qs


def test_audit_matches_reference_count(case):
    w, ref, eng, qs = case
    got = eng.audit_ub(0, qs, 1e-6)
    assert got == ref.audit(qs, 1e-6) == 0  # a built index is sound (acceptance C1)


def _file_bytes(ix, cfg, keys, values, texts):
    """save_index layout (serialize.cpp:127-148) built from our codec + the store."""
    out = bytearray(api.index_to_bytes(ix, cfg))
    n, d = keys.shape
    out += n.to_bytes(8, "little")
    for t in texts:
        b = t.encode()
        out += len(b).to_bytes(8, "little") + b
    for a in (keys, values):
        out += (n * d).to_bytes(8, "little") + np.ascontiguousarray(a, np.float32).tobytes()
    return bytes(out)


def test_audit_flags_shrunken_radii(case, tmp_path):
    """test_evaluator.cpp:146-173: shrinking radii must be flagged -- the device
    count equals the reference's on the same (modified) index."""
    w, ref, eng, qs = case
    ix = host_index(ref)
    ix.fine_radius = ix.fine_radius * 0.5
    ix.coarse_radius = ix.coarse_radius * 0.9
    eng2 = api.Engine(1, 128, 4, cap_tokens=8192 + 64, cap_chunks=2048, cap_clusters=1024, cap_units=64)
    eng2.upload_slot(0, ix, w.keys, w.values)
    texts = ["\n" if c == 1 else ("}" if c == 2 else "") for c in w.text_code]
    p = tmp_path / "shrunk.tkix"
    p.write_bytes(_file_bytes(ix, api.IndexConfig(seed=31), w.keys, w.values, texts))
    bad = R.RefEngine.load(str(p))
    for tol in (1e-6, 0.05):
        exp = bad.audit(qs, tol)
        assert exp > 0
        assert eng2.audit_ub(0, qs, tol) == exp


def test_oracle_topk_matches_reference(case):
    w, ref, eng, qs = case
    for budget in (1, 64, 2048, 100000):
        got = eng.oracle_topk(0, qs[:6], budget)
        for i in range(6):
            exp = ref.oracle_topk(qs[i], budget)
            assert np.array_equal(got[i], exp), (budget, i)


def test_oracle_topk_ties_go_to_smaller_ids():
    # duplicate keys: equal scores must resolve toward the smaller token id
    rng = np.random.default_rng(2)
    base = api.bf16_round(rng.standard_normal((64, 128)).astype(np.float32))
    keys = np.concatenate([base] * 8)
    w = rounded_workload(512, 128, seed=3, n_blobs=2, query_count=2)
    ref = R.RefEngine(keys, w.values, w.text_code, seed=3)
    eng = api.Engine(1, 128, 2, cap_tokens=600, cap_chunks=200, cap_clusters=100, cap_units=16)
    eng.upload_slot(0, host_index(ref), keys, w.values)
    q = rng.standard_normal((3, 128)).astype(np.float32)
    got = eng.oracle_topk(0, q, 100)
    for i in range(3):
        assert np.array_equal(got[i], ref.oracle_topk(q[i], 100))


def test_full_attention_matches_reference(case):
    w, ref, eng, qs = case
    q = torch.from_numpy(np.ascontiguousarray(w.queries)).cuda()
    out = eng.full_attention(0, q).cpu().numpy()
    for g in range(4):
        assert rel_l2(out[g], ref.full_attention(w.queries[g])) < 1e-3
    with pytest.raises(api.L.LcError):
        eng.oracle_topk(0, qs[:1], 0)  # oracle_topk_tokens: budget >= 1


def test_audit_after_device_grafts_is_sound():
    """acceptance C1's second half: grafts keep the index sound (device grafts,
    audited on the device, cross-checked by the reference after the same grafts)."""
    w = rounded_workload(3000, 128, seed=4, n_blobs=3, query_count=2)
    ref = R.RefEngine(w.keys, w.values, w.text_code, seed=4)
    texts = ["\n" if c == 1 else ("}" if c == 2 else "") for c in w.text_code]
    st = api.StreamState(host_index(ref), w.keys, w.values, texts)
    rng = np.random.default_rng(9)
    n0 = w.keys.shape[0]
    for i in range(400):
        k = api.bf16_round(rng.standard_normal(128).astype(np.float32))
        k = api.bf16_round(k / np.linalg.norm(k))
        v = api.bf16_round(rng.standard_normal(128).astype(np.float32))
        ref.push_and_graft(k, v, 0)
        st.push_token(n0 + i, "", k, v)
    qs = rng.standard_normal((64, 128)).astype(np.float32)
    assert st.engine.audit_ub(0, qs, 1e-6) == ref.audit(qs, 1e-6) == 0
