"""The fused all-gather epilogue (lc_set_gather / lc_gather_wait) on one GPU:
two "peer" gather buffers and arrival counters in local memory stand in for
two ranks' NVLink peer memory.  Every merged (slot, head) row must land at its
row in both buffers, each counter must advance by exactly one per row, and
the wait must release -- eagerly, per layer (lc_retrieve_slots), and inside a
CUDA graph replayed several times."""
import numpy as np
import pytest

from paper_2603_08453_b200 import api

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _engine(S=6, G=4, n=8192):
    cap_chunks = n // 8 + 64
    eng = api.Engine(S, 128, G, cap_tokens=n + 64, cap_chunks=cap_chunks, cap_clusters=(cap_chunks + 1) // 2,
                     cap_units=64)
    seeds = np.arange(700, 700 + S, dtype=np.uint64)
    codes, qs = eng.gen_workload(n, seeds, query_count=G)
    eng.build_index([n] * S, [api.segment_codes(codes[s]) for s in range(S)], seeds)
    return eng, torch.from_numpy(qs).cuda()


def test_fused_gather_local_peers_eager_layerwise_and_graph():
    S, G = 6, 4
    eng, q = _engine(S, G)
    b = api.Budgets(token_budget=1024)
    out = torch.zeros_like(q)
    bufs = [torch.full((S, G, 128), -1.0, device="cuda") for _ in range(2)]
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    rows = np.arange(S)[::-1].copy()  # a permutation: slot s -> row S-1-s
    fptr = [flags.data_ptr(), flags.data_ptr() + 4]
    eng.set_gather([x.data_ptr() for x in bufs], fptr, rows, fptr[0], S * G)
    for _ in range(3):
        eng.retrieve(q, b, out=out)
        eng.gather_wait()
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    for x in bufs:
        assert np.array_equal(x.cpu().numpy()[rows], o)
    assert flags.cpu().tolist() == [3 * S * G, 3 * S * G]
    assert eng.device_error() == 0

    # layer by layer: two "layers" of 3 slots, one wait per layer
    eng.set_gather([x.data_ptr() for x in bufs], fptr, rows, fptr[0], 3 * G)
    flags.zero_()
    for x in bufs:
        x.fill_(-1.0)
    for layer in range(2):
        eng.retrieve_slots(3 * layer, 3, q, b, out=out)
        eng.gather_wait()
    torch.cuda.synchronize()
    for x in bufs:
        assert np.array_equal(x.cpu().numpy()[rows], out.cpu().numpy())
    assert flags.cpu().tolist() == [S * G, S * G]

    # captured: retrieve + wait replayed three times
    eng.set_gather([x.data_ptr() for x in bufs], fptr, rows, fptr[0], S * G)
    flags.zero_()
    eng.retrieve(q, b, out=out)
    eng.gather_wait()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cs):
        eng.retrieve(q, b, out=out)
        eng.gather_wait()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert flags.cpu().tolist() == [4 * S * G, 4 * S * G]
    for x in bufs:
        assert np.array_equal(x.cpu().numpy()[rows], out.cpu().numpy())
    assert eng.device_error() == 0
    eng.set_gather([], [], [], 0, 0)
    with pytest.raises(Exception):
        eng.gather_wait()
