"""lc_retrieve_slots (one layer's slots of a layer-by-layer decode) gives the
same selections as one lc_retrieve over every slot (bit-exact) and the same
outputs up to fp32 merge order (the persistent attention kernel cuts the
launched slots' token sequence into different warp ranges, so the partials
combine in a different order), and leaves the rows outside its range
untouched."""
import numpy as np
import pytest

from paper_2603_08453_b200 import api

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_retrieve_slots_equals_full_launch():
    n, S, G = 8192, 6, 4
    cap_chunks = n // 8 + 64
    eng = api.Engine(S, 128, G, cap_tokens=n + 64, cap_chunks=cap_chunks, cap_clusters=(cap_chunks + 1) // 2,
                     cap_units=64)
    seeds = np.arange(500, 500 + S, dtype=np.uint64)
    codes, qs = eng.gen_workload(n, seeds, query_count=G)
    eng.build_index([n] * S, [api.segment_codes(codes[s]) for s in range(S)], seeds)
    q = torch.from_numpy(qs).cuda()
    b = api.Budgets(token_budget=1024)
    full = torch.zeros_like(q)
    eng.retrieve(q, b, out=full)
    ref_sel = [[eng.selection(s, g) for g in range(G)] for s in range(S)]
    part = torch.full_like(q, 7.0)
    for first, count in ((0, 2), (2, 3), (5, 1)):
        eng.retrieve_slots(first, count, q, b, out=part)
        torch.cuda.synchronize()
        p = part.cpu().numpy()
        f = full.cpu().numpy()[first:first + count]
        assert np.abs(p[first:first + count] - f).max() <= 1e-5 * np.abs(f).max()
        assert (p[first + count:] == 7.0).all()
        for s in range(first, first + count):
            for g in range(G):
                got = eng.selection(s, g)
                assert np.array_equal(got.selected_clusters, ref_sel[s][g].selected_clusters)
                assert np.array_equal(got.active_token_ids, ref_sel[s][g].active_token_ids)
    with pytest.raises(Exception):
        eng.retrieve_slots(5, 2, q, b, out=part)
    assert eng.device_error() == 0
