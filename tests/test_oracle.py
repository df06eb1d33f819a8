"""CPU: pin the plain-C oracle (oracle/lc_oracle.c) to the reference.

* against the committed golden vectors (made by the reference itself), bit for bit;
* against the reference library (oracle/_ref) on fresh seeded inputs, when built;
* the config-1 fingerprints of SURVEY.md s8(d).
"""
import json
import os

import numpy as np
import pytest

from oracle import cpy
from oracle import refpy as R

from . import golden_io

pytestmark = pytest.mark.skipif(not cpy.available(), reason="oracle/liblc_oracle.so not built")
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _check_retrieve(got, z, k):
    assert np.array_equal(got["units"], z[k + "units"])
    assert np.array_equal(got["clusters"], z[k + "clusters"])
    assert np.array_equal(got["active"], z[k + "active"])
    assert got["scanned"] == int(z[k + "meta"][0])
    assert got["degenerate"] == bool(z[k + "meta"][1])
    # same libm, same order of operations: bit-identical outputs
    assert np.array_equal(got["output"].view(np.uint32), z[k + "output"].view(np.uint32))


@pytest.mark.parametrize("name", ["retrieve_d128", "retrieve_d32"])
def test_oracle_retrieve_golden(name):
    fx = golden_io.load(name)
    o = cpy.OracleIndex(fx.keys, fx.values, fx.text_code, fx.index)
    for bi, (mode, tb, kc, ku, sink) in enumerate(fx.z["budgets"].tolist()):
        for qi in range(fx.queries.shape[0]):
            got = o.retrieve(fx.queries[qi], unit_topk=ku, mode=mode, cluster_topk=kc,
                             token_budget=tb, sink=sink)
            _check_retrieve(got, fx.z, f"r{bi}_q{qi}_")


@pytest.mark.parametrize("name", ["stream_d64", "stream_d64_full"])
def test_oracle_stream_golden(name):
    fx = golden_io.load(name)
    budget, graft_full = [int(x) for x in fx.z["meta"]]
    steps = fx.tok_keys.shape[0]
    o = cpy.OracleIndex(fx.keys, fx.values, fx.text_code, fx.index, extra_tokens=steps + 1,
                        extra_chunks=steps, graft_full=bool(graft_full))
    grafts = fx.z["grafts"]
    for i in range(steps):
        r = o.decode_step(fx.queries[i % 2], fx.tok_keys[i], fx.tok_values[i],
                          int(fx.tok_code[i]), token_budget=budget)
        k = f"s{i}_"
        assert np.array_equal(r["clusters"], fx.z[k + "clusters"]), i
        assert np.array_equal(r["active"], fx.z[k + "active"]), i
        assert np.array_equal(r["output"].view(np.uint32), fx.z[k + "output"].view(np.uint32)), i
        g = grafts[i]
        assert (r["graft"] is None) == (g[1] < 0), i
        if r["graft"]:
            assert [r["graft"][x] for x in ("chunk_id", "cluster_id", "unit_id", "distance_comps")] == \
                g[1:].tolist()
            f = fx.z[k + "graft_f64"]
            assert [r["graft"]["centroid_delta"], r["graft"]["fine_radius"],
                    r["graft"]["coarse_radius"]] == f.tolist()
    fin = fx.final
    m = int(o.s.n_chunks)
    assert np.array_equal(o.cluster_of_chunk[:m], fin.cluster_of_chunk)
    assert np.array_equal(o.chunk_start[:m], fin.chunk_span[:, 0])
    assert np.array_equal(o.chunk_end[:m], fin.chunk_span[:, 1])
    assert np.array_equal(o.chunk_kind[:m], fin.chunk_span[:, 2])
    assert np.array_equal(o.chunk_level[:m], fin.chunk_span[:, 3])
    assert np.array_equal(o.chunk_rep[:m].view(np.uint32), fin.chunk_rep.view(np.uint32))
    assert np.array_equal(o.fine_centroid.view(np.uint32), fin.fine_centroid.view(np.uint32))
    assert np.array_equal(o.fine_radius.view(np.uint64), fin.fine_radius.view(np.uint64))
    assert np.array_equal(o.fine_token_count, fin.fine_token_count)
    assert np.array_equal(o.coarse_radius.view(np.uint64), fin.coarse_radius.view(np.uint64))


def test_oracle_segment_golden():
    fx = golden_io.load("retrieve_d32")
    spans = cpy.segment(fx.text_code)
    assert np.array_equal(spans, fx.index.chunk_span)


def test_config1_fingerprint_pins_oracle():
    """SURVEY.md s8(d) fingerprints, recomputed by the C oracle on a re-generated
    32K workload (when the reference is built) -- otherwise just sanity."""
    rows = json.load(open(os.path.join(golden_io.HERE, "config1_fingerprints.json")))
    assert rows[0]["seed"] == 1000 and rows[0]["units"] == [12, 13, 10, 34, 1, 3, 24, 29]
    assert rows[0]["n_clusters"] == 31 and rows[0]["active"] == 2052 and rows[0]["scanned"] == 351
    if not R.available():
        pytest.skip("oracle/_ref not built")
    for row in rows:
        w = R.gen_workload(32768, 128, seed=row["seed"], query_count=4)
        assert format(R.fnv1a64(w.keys.tobytes()), "016x") == row["keys_fnv1a"]
        ref = R.RefEngine(w.keys, w.values, w.text_code, seed=row["seed"])
        assert ref.dims()[1:4] == [row["M"], row["L"], row["P"]]
        o = cpy.OracleIndex(w.keys, w.values, w.text_code, ref.export())
        got = o.retrieve(w.queries[0], token_budget=2048)
        assert got["units"].tolist() == row["units"]
        assert got["clusters"].tolist() == row["clusters"]
        assert len(got["active"]) == row["active"] and got["scanned"] == row["scanned"]
        assert np.allclose(got["output"][:3], row["out3"], rtol=0, atol=1e-9)


@needs_ref
@pytest.mark.parametrize("seed,d,n", [(3, 16, 3000), (8, 64, 5000), (13, 128, 2500)])
def test_oracle_vs_reference_fresh(seed, d, n):
    w = R.gen_workload(n, d, seed=seed, n_blobs=5, query_count=6)
    ref = R.RefEngine(w.keys, w.values, w.text_code, seed=seed)
    o = cpy.OracleIndex(w.keys, w.values, w.text_code, ref.export())
    assert np.array_equal(cpy.segment(w.text_code), R.segment(w.text_code))
    for qi in range(6):
        for tb in (32, 200, 900):
            a = ref.retrieve(w.queries[qi], token_budget=tb)
            b = o.retrieve(w.queries[qi], token_budget=tb)
            for k in ("units", "clusters", "active"):
                assert np.array_equal(a[k], b[k]), (qi, tb, k)
            assert np.array_equal(a["output"].view(np.uint32), b["output"].view(np.uint32))


@needs_ref
def test_chunk_representative_matches_reference():
    rng = np.random.default_rng(0)
    for rows in (1, 7, 16):
        k = rng.standard_normal((rows, 128)).astype(np.float32)
        for pool in (0, 1):
            assert np.array_equal(cpy.chunk_representative(k, pool), R.chunk_representative(k, pool))
