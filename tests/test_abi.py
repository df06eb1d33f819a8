"""CPU: the C-ABI library loads, exports every declared symbol, and its host
logic (chunker, flush decision, argument validation) behaves like the reference."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import cpy
from paper_2603_08453_b200 import _lib, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lychee_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(lc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert sorted(_lib.EXPORTS) == names


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(_lib.LcError):
        api.Engine(1, 128, 4, cap_tokens=64, cap_chunks=8, cap_clusters=8, cap_units=4)


def test_create_validates_shape():
    d = _lib.IndexDesc(1, 96, 4, 64, 8, 8, 4, 0, 0, 1, 0, 1, 0, 0, 0)
    h = C.c_void_p()
    assert _lib.lib().lc_index_create(C.byref(d), C.byref(h)) == _lib.LC_EINVAL
    d = _lib.IndexDesc(1, 128, 9, 64, 8, 8, 4, 0, 0, 1, 0, 1, 0, 0, 0)
    assert _lib.lib().lc_index_create(C.byref(d), C.byref(h)) == _lib.LC_EINVAL
    assert b"group" in _lib.lib().lc_last_error()


def test_segment_matches_oracle_on_planted_markers():
    rng = np.random.default_rng(1)
    for n in (1, 7, 8, 9, 16, 17, 100, 1000):
        codes = (rng.random(n) < 0.1).astype(np.uint8) + ((rng.random(n) < 0.03) * 2).astype(np.uint8)
        codes = np.minimum(codes, 2)
        texts = ["\n" if c == 1 else ("}" if c == 2 else "") for c in codes]
        assert np.array_equal(api.segment(texts), cpy.segment(codes)), n


def test_segment_text_levels():
    # chunker KATs in the spirit of test_chunker.cpp: strongest separator wins,
    # rightmost among equal levels, spanning "\n\n" is level 1
    texts = ["a"] * 20
    texts[9] = "x,"
    texts[11] = "y."
    sp = api.segment(texts)
    assert sp[0].tolist() == [0, 12, 0, 2]
    texts = ["a"] * 20
    texts[9], texts[10] = "\n", "\n"
    assert api.segment(texts)[0].tolist() == [0, 11, 0, 1]
    texts = ["w "] * 16
    assert api.segment(texts)[0].tolist() == [0, 16, 0, 4]
    assert api.segment(["a"] * 5)[0].tolist() == [0, 5, 2, 0]
    with pytest.raises(_lib.LcInvalidArgument):
        api.segment([])


def test_flush_take_matches_streamer_rules():
    # streamer test KATs (test_streamer.cpp:91-116)
    assert api.flush_take([""] * 16) == (16, 1, 0)
    texts = [""] * 16
    texts[10] = "}"
    assert api.flush_take(texts) == (11, 0, 1)
    assert api.flush_take(texts, structure_aware=False) == (16, 1, 0)


def test_budgets_validate():
    with pytest.raises(ValueError):
        api.Budgets(unit_topk=0).validate()
    with pytest.raises(ValueError):
        api.Budgets(token_budget=0).validate()
    with pytest.raises(ValueError):
        api.Budgets(mode=api.SelectionMode.fixed_cluster_count, cluster_topk=0).validate()
    api.Budgets().validate()


def test_bf16_rounding_is_nearest_even():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.1415927, 1e-30, 65504.0], np.float32)
    torch = pytest.importorskip("torch")
    expect = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(api.bf16_round(x), expect)
