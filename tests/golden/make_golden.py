"""Generate the committed golden vectors from the reference itself.

Run in the build container (needs oracle/_ref, i.e. /root/reference compiled
by `make -C oracle ref`):  python tests/golden/make_golden.py

Every fixture stores bf16-rounded K/V (as bf16 bit patterns), the reference's
HierarchicalIndex built on them by the reference's build_index, the queries,
and the reference's outputs (retrieve / decode_step / graft reports / final
index), so the C oracle and the device path can be pinned without the
reference on the GPU box.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refpy as R  # noqa: E402
from paper_2603_08453_b200.api import bf16_bits, bf16_round  # noqa: E402

IDX_FIELDS = ("chunk_span", "chunk_rep", "fine_centroid", "fine_radius", "fine_token_count",
              "fine_parent", "fine_member_off", "fine_members", "coarse_centroid", "coarse_radius",
              "coarse_member_off", "coarse_members", "cluster_of_chunk")

BUDGETS = [  # (mode, token_budget, cluster_topk, unit_topk, sink)
    (1, 64, 8, 8, 16), (1, 256, 8, 8, 16), (1, 1024, 8, 8, 16), (1, 256, 8, 3, 0),
    (0, 1024, 1, 8, 16), (0, 1024, 8, 8, 16), (0, 1024, 37, 8, 16),
]


def export_dict(e: R.IndexExport, prefix="ix_"):
    return {prefix + f: getattr(e, f) for f in IDX_FIELDS}


def retrieve_fixture(name, n, d, seed, n_blobs, nq):
    w = R.gen_workload(n, d, seed=seed, n_blobs=n_blobs, query_count=nq)
    keys, values = bf16_round(w.keys), bf16_round(w.values)
    ref = R.RefEngine(keys, values, w.text_code, seed=seed)
    out = dict(keys_bf16=bf16_bits(keys), values_bf16=bf16_bits(values), text_code=w.text_code,
               queries=w.queries, budgets=np.array(BUDGETS, np.uint64))
    out.update(export_dict(ref.export()))
    for bi, (mode, tb, kc, ku, sink) in enumerate(BUDGETS):
        for qi in range(nq):
            r = ref.retrieve(w.queries[qi], unit_topk=ku, mode=mode, cluster_topk=kc,
                             token_budget=tb, sink=sink)
            k = f"r{bi}_q{qi}_"
            out[k + "units"] = r["units"]
            out[k + "clusters"] = r["clusters"]
            out[k + "active"] = r["active"]
            out[k + "output"] = r["output"]
            out[k + "meta"] = np.array([r["scanned"], int(r["degenerate"])], np.uint64)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def stream_tokens(centers, steps, d, seed):
    rng = np.random.default_rng(seed)
    ks, vs, codes = [], [], []
    for i in range(steps):
        c = centers[rng.integers(len(centers))]
        k = c + 0.1 * rng.standard_normal(d)
        ks.append((k / np.linalg.norm(k)).astype(np.float32))
        vs.append(rng.standard_normal(d).astype(np.float32))
        codes.append(1 if i % 12 == 7 else (2 if i % 29 == 3 else 0))
    return bf16_round(np.array(ks)), bf16_round(np.array(vs)), np.array(codes, np.uint8)


def stream_fixture(name, n, d, seed, steps, budget, graft_full):
    w = R.gen_workload(n, d, seed=seed, n_blobs=3, query_count=2)
    keys, values = bf16_round(w.keys), bf16_round(w.values)
    ref = R.RefEngine(keys, values, w.text_code, seed=seed, graft_full=graft_full)
    out = dict(keys_bf16=bf16_bits(keys), values_bf16=bf16_bits(values), text_code=w.text_code,
               queries=w.queries, meta=np.array([budget, int(graft_full)], np.uint64))
    out.update(export_dict(ref.export()))
    ks, vs, codes = stream_tokens(w.centers, steps, d, seed + 7)
    out["tok_keys_bf16"], out["tok_values_bf16"], out["tok_code"] = bf16_bits(ks), bf16_bits(vs), codes
    grafts = []
    for i in range(steps):
        r = ref.decode_step(w.queries[i % 2], ks[i], vs[i], int(codes[i]), token_budget=budget)
        k = f"s{i}_"
        out[k + "clusters"] = r["clusters"]
        out[k + "active"] = r["active"]
        out[k + "output"] = r["output"]
        out[k + "meta"] = np.array([r["scanned"], int(r["degenerate"])], np.uint64)
        out[k + "stab"] = np.array([r["jaccard"], r["window_hit"]], np.float64)
        g = r["graft"]
        grafts.append([i, g["chunk_id"], g["cluster_id"], g["unit_id"], g["distance_comps"]]
                      if g else [i, -1, -1, -1, -1])
        if g:
            out[k + "graft_f64"] = np.array([g["centroid_delta"], g["fine_radius"],
                                             g["coarse_radius"]], np.float64)
    out["grafts"] = np.array(grafts, np.int64)
    out.update(export_dict(ref.export(), "final_"))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


# SURVEY.md s8(d) lists these for seeds 1002..1007 (measured with the reference
# while surveying): n_clusters, active, scanned of query 0
SURVEY_Q0 = {1002: (41, 2048, 429), 1003: (43, 2035, 468), 1004: (36, 2006, 443),
             1005: (36, 2037, 698), 1006: (31, 2044, 220), 1007: (44, 2056, 474)}


def fingerprints():
    """Config-1 fingerprints: 32K tokens, d=128, 4 queries (one
    GQA group) per KV head, B=2048, seeds 1000..1007 = the 8 KV heads of one layer.
    Top-level fields describe query 0 (the SURVEY table); `heads` holds all 4."""
    rows = []
    for seed in range(1000, 1008):
        w = R.gen_workload(32768, 128, seed=seed, query_count=4)
        ref = R.RefEngine(w.keys, w.values, w.text_code, seed=seed)
        dims = ref.dims()
        heads = []
        for g in range(4):
            r = ref.retrieve(w.queries[g], token_budget=2048)
            heads.append(dict(units=r["units"].tolist(), clusters=r["clusters"].tolist(),
                              active=len(r["active"]), scanned=r["scanned"],
                              out3=[float(x) for x in r["output"][:3]]))
        h0 = heads[0]
        if seed in SURVEY_Q0:
            assert (len(h0["clusters"]), h0["active"], h0["scanned"]) == SURVEY_Q0[seed], seed
        rows.append(dict(seed=seed, M=dims[1], L=dims[2], P=dims[3],
                         keys_fnv1a=format(R.fnv1a64(w.keys.tobytes()), "016x"),
                         units=h0["units"], n_clusters=len(h0["clusters"]), first5=h0["clusters"][:5],
                         active=h0["active"], scanned=h0["scanned"], out3=h0["out3"],
                         clusters=h0["clusters"], heads=heads))
    with open(os.path.join(HERE, "config1_fingerprints.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    import sys
    if sys.argv[1:] == ["fingerprints"]:
        fingerprints()
        sys.exit(0)
    retrieve_fixture("retrieve_d128", 1200, 128, seed=21, n_blobs=4, nq=4)
    retrieve_fixture("retrieve_d32", 4096, 32, seed=21, n_blobs=4, nq=4)
    stream_fixture("stream_d64", 800, 64, seed=4, steps=160, budget=128, graft_full=False)
    stream_fixture("stream_d64_full", 800, 64, seed=5, steps=96, budget=128, graft_full=True)
    fingerprints()
    print("golden fixtures written to", HERE)
