"""Config 3 (streaming decode with lazy grafts) on the GPU.

* lc_decode_step_async (device take / kind / level, no host sync, graph-
  capturable) produces the same selections, outputs, graft reports and final
  index as the host-synchronous lc_decode_step, eagerly and inside one CUDA
  graph of many steps.
* At config 3's per-slot scale -- a 128K GPU-built prefix, then 4096 decoded
  tokens -- every sampled step's selection, every graft report and the final
  index_to_bytes stream equal the reference's own StreamState::decode_step
  (streamer.cpp:145-165) driven with the same tokens.
* The device-side checks that replace the host ones raise their error bits.
"""
import os

import numpy as np
import pytest

from oracle import refpy as R
from paper_2603_08453_b200 import api

from ._helpers import assert_same_selection, rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
TOL = 1e-3
ERR_TAKE = 1 << 7


def texts_of(codes):
    return ["\n" if c == 1 else ("}" if c == 2 else "") for c in codes]


def _gpu_engine(n, seeds, G, extra, keep_reps=True):
    S = len(seeds)
    cap_chunks = n // 8 + 64 + extra // 8 + 8
    eng = api.Engine(S, 128, G, cap_tokens=n + extra + 64, cap_chunks=cap_chunks,
                     cap_clusters=(n // 8 + 65) // 2, cap_units=64, keep_reps=keep_reps)
    codes, qs = eng.gen_workload(n, np.array(seeds, np.uint64), query_count=G)
    spans = [api.segment_codes(codes[s]) for s in range(S)]
    eng.build_index([n] * S, spans, seeds)
    return eng, codes, qs


def _tokens(qs, steps, seed):
    """run_stream-style decoded tokens (bench.cpp:240-272): stationary queries
    around each slot's own queries, unit keys near them, N(0,1) values, a
    newline marker every 12 steps; bf16-rounded so both sides see the same
    values."""
    rng = np.random.default_rng(seed)
    S, G, d = qs.shape
    out = []
    for i in range(steps):
        q = qs + 0.05 * rng.standard_normal(qs.shape)
        q = (q * (np.sqrt(d) / np.linalg.norm(q, axis=-1, keepdims=True))).astype(np.float32)
        k = qs[:, 0] / np.sqrt(d) + 0.1 * rng.standard_normal((S, d))
        k = api.bf16_round((k / np.linalg.norm(k, axis=-1, keepdims=True)).astype(np.float32))
        v = api.bf16_round(rng.standard_normal((S, d)).astype(np.float32))
        out.append((q, k, v, 1 if (i + 1) % 12 == 0 else 0))
    return out


class _Chunker:
    """The host flush decision (streamer.cpp:29-66) over the shared text stream."""

    def __init__(self):
        self.buf = []

    def push(self, code):
        self.buf.append("\n" if code == 1 else "")
        if len(self.buf) < 16:
            return None
        t, kd, lv = api.flush_take(self.buf)
        self.buf = self.buf[t:]
        return t, kd, lv


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _bits(k):
    return _dev(api.bf16_bits(k).view(np.int16))


def test_async_matches_sync_eager_and_graph():
    n, seeds, G, steps = 8192, [31, 32, 33], 4, 120
    toks = None
    results = {}
    for mode in ("sync", "async", "graph"):
        eng, codes, qs = _gpu_engine(n, seeds, G, steps)
        if toks is None:
            toks = _tokens(qs, steps, 5)
        S = len(seeds)
        b = api.Budgets(token_budget=512)
        ch = _Chunker()
        plan = [ch.push(code) for *_, code in toks]
        outs = torch.zeros((steps, S, G, 128), device="cuda")
        qd = [_dev(q) for q, *_ in toks]
        kd = [(_bits(k), _bits(v)) for _, k, v, _ in toks]
        tk = [None if p is None else tuple(_dev(np.full(S, x, np.uint32)) for x in p) for p in plan]
        reps = []
        if mode == "sync":
            for i in range(steps):
                p = plan[i]
                args = (None, None, None) if p is None else tuple(np.full(S, x, np.uint32) for x in p)
                eng.decode_step(qd[i], kd[i][0], kd[i][1], b, *args, out=outs[i])
                if p is not None:
                    reps.append(eng.reports().copy())
        elif mode == "async":
            for i in range(steps):
                t = tk[i] or (None, None, None)
                eng.decode_step_async(qd[i], kd[i][0], kd[i][1], b, *t, out=outs[i])
                if plan[i] is not None:
                    reps.append(eng.reports().copy())
        else:
            # warm-up (scratch allocation) outside the graph, then the rest in one graph
            eng.decode_step_async(qd[0], kd[0][0], kd[0][1], b, *(tk[0] or (None,) * 3), out=outs[0])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=cs):
                for i in range(1, steps):
                    eng.decode_step_async(qd[i], kd[i][0], kd[i][1], b, *(tk[i] or (None,) * 3), out=outs[i])
            g.replay()
            torch.cuda.synchronize()
        assert eng.device_error() == 0, mode
        results[mode] = (outs.cpu().numpy(), [eng.index_bytes(s) for s in range(S)], reps,
                         [eng.slot_dims(s) for s in range(S)])
        del eng
        torch.cuda.empty_cache()
    assert sum(p is not None for p in plan) >= 6
    for mode in ("async", "graph"):
        assert np.array_equal(results[mode][0], results["sync"][0]), mode
        assert results[mode][1] == results["sync"][1], mode
        assert results[mode][3] == results["sync"][3], mode
    assert len(results["async"][2]) == len(results["sync"][2])
    for a, s in zip(results["async"][2], results["sync"][2]):
        assert a.tobytes() == s.tobytes()


def test_async_take_checked_on_device():
    """take larger than the buffered tokens: the graft kernel refuses it (error
    bit) instead of grafting past the store, and the index is unchanged."""
    eng, codes, qs = _gpu_engine(4096, [41], 4, 64)
    b = api.Budgets(token_budget=512)
    before = eng.index_bytes(0)
    k = _bits(api.bf16_round(np.ones((1, 128), np.float32) / np.sqrt(128)))
    take = _dev(np.array([40], np.uint32))
    eng.decode_step_async(_dev(qs), k, k, b, take, None, None, out=torch.zeros((1, 4, 128), device="cuda"))
    assert eng.device_error() & ERR_TAKE
    assert eng.slot_dims(0)[4] == 4097  # the token was appended
    assert eng.index_bytes(0) == before


@pytest.mark.parametrize("seed", [1300])
def test_config3_stream_parity_at_scale(tmp_path, seed):
    """A config-3 slot: 128K GPU-built prefix, then 4096 decode steps through
    lc_decode_step_async; the reference StreamState (loaded from the GPU
    slot's TKIX file) decodes the same tokens.  Every 64th step's selection and
    output, every graft report and the final index bytes must match."""
    n, steps, G = 131072, 4096, 1
    eng, codes, qs = _gpu_engine(n, [seed], G, steps)
    p = str(tmp_path / "slot.tkix")
    eng.save_index(0, p, texts_of(codes[0]))
    ref = R.RefEngine.load(p)
    os.remove(p)
    assert ref.index_bytes() == eng.index_bytes(0)
    toks = _tokens(qs, steps, 9)
    b = api.Budgets(token_budget=2048)
    ch = _Chunker()
    out = torch.zeros((1, G, 128), device="cuda")
    grafts = 0
    for i, (q, k, v, code) in enumerate(toks):
        plan = ch.push(code)
        t = (None, None, None) if plan is None else tuple(_dev(np.array([x], np.uint32)) for x in plan)
        eng.decode_step_async(_dev(q), _bits(k), _bits(v), b, *t, out=out)
        r = ref.decode_step(q[0, 0], k[0], v[0], code, token_budget=2048)
        assert (plan is None) == (r["graft"] is None), i
        if plan is not None:
            grafts += 1
            rep = eng.reports()[0]
            g = r["graft"]
            assert (int(rep["chunk_id"]), int(rep["cluster_id"]), int(rep["unit_id"]),
                    int(rep["distance_comps"])) == (g["chunk_id"], g["cluster_id"], g["unit_id"],
                                                    g["distance_comps"]), i
            assert float(rep["centroid_delta"]) == g["centroid_delta"], i
            assert float(rep["fine_radius"]) == g["fine_radius"], i
            assert float(rep["coarse_radius"]) == g["coarse_radius"], i
        if i % 64 == 63:
            got = eng.selection(0, 0)
            assert_same_selection(got, r, i)
            assert rel_l2(out.cpu().numpy()[0, 0], r["output"]) < TOL, i
    assert grafts >= 4096 // 16
    assert eng.device_error() == 0
    assert eng.slot_dims(0)[4] == n + steps
    assert eng.index_bytes(0) == ref.index_bytes()


def test_compaction_keeps_selections_and_index():
    """lc_compact folds the grafted chunks into the member CSR: the next
    retrieve selects the same clusters and active ids, the index bytes are
    unchanged, and further grafts keep matching the uncompacted twin."""
    n, seeds, G, steps = 8192, [61, 62], 4, 200
    engs = []
    for _ in range(2):
        eng, codes, qs = _gpu_engine(n, seeds, G, steps + 64)
        engs.append(eng)
    toks = _tokens(qs, steps, 3)
    b = api.Budgets(token_budget=512)
    ch = _Chunker()
    S = len(seeds)
    out = [torch.zeros((S, G, 128), device="cuda") for _ in engs]
    for i, (q, k, v, code) in enumerate(toks):
        plan = ch.push(code)
        t = (None, None, None) if plan is None else tuple(_dev(np.full(S, x, np.uint32)) for x in plan)
        for e, o in zip(engs, out):
            e.decode_step_async(_dev(q), _bits(k), _bits(v), b, *t, out=o)
        if i in (99, 150):
            engs[0].compact(1)  # engine 0 compacts explicitly (engine 1 only by the every-128-steps rule)
        if i % 25 == 24:
            for s in range(S):
                for g in range(G):
                    a0, a1 = engs[0].selection(s, g), engs[1].selection(s, g)
                    assert np.array_equal(a0.selected_clusters, a1.selected_clusters), (i, s, g)
                    assert np.array_equal(a0.active_token_ids, a1.active_token_ids), (i, s, g)
            assert np.array_equal(out[0].cpu().numpy(), out[1].cpu().numpy()), i
    for s in range(S):
        assert engs[0].index_bytes(s) == engs[1].index_bytes(s)
    assert all(e.device_error() == 0 for e in engs)
