"""Loader for the committed golden vectors (tests/golden/*.npz, made by
tests/golden/make_golden.py from the reference itself)."""
from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
IDX_FIELDS = ("chunk_span", "chunk_rep", "fine_centroid", "fine_radius", "fine_token_count",
              "fine_parent", "fine_member_off", "fine_members", "coarse_centroid", "coarse_radius",
              "coarse_member_off", "coarse_members", "cluster_of_chunk")


def widen(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _index(z, prefix):
    ns = SimpleNamespace(**{f: z[prefix + f] for f in IDX_FIELDS})
    ns.dim = int(ns.fine_centroid.shape[1])
    return ns


def load(name: str):
    z = np.load(os.path.join(HERE, name + ".npz"))
    fx = SimpleNamespace(z=z)
    fx.keys = widen(z["keys_bf16"])
    fx.values = widen(z["values_bf16"])
    fx.text_code = z["text_code"]
    fx.queries = z["queries"]
    fx.index = _index(z, "ix_")
    if "final_chunk_span" in z.files:
        fx.final = _index(z, "final_")
    if "tok_keys_bf16" in z.files:
        fx.tok_keys = widen(z["tok_keys_bf16"])
        fx.tok_values = widen(z["tok_values_bf16"])
        fx.tok_code = z["tok_code"]
    return fx
