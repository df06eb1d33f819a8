"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/liblc_oracle.so`` (the plain-C restatement in
``lc_oracle.c``).  ``OracleIndex`` owns numpy buffers laid out as ``lco_index``
(orig numbering, exactly the reference's fields) and is populated from a
reference ``IndexExport`` or from the golden fixtures.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblc_oracle.so")

_lib = None


class LcoIndex(C.Structure):
    _fields_ = [
        ("d", C.c_uint32), ("n_tokens", C.c_uint32), ("cap_tokens", C.c_uint32),
        ("chunked_end", C.c_uint32),
        ("keys", C.c_void_p), ("values", C.c_void_p), ("text_code", C.c_void_p),
        ("n_chunks", C.c_uint32), ("cap_chunks", C.c_uint32),
        ("chunk_start", C.c_void_p), ("chunk_end", C.c_void_p), ("chunk_kind", C.c_void_p),
        ("chunk_level", C.c_void_p), ("chunk_rep", C.c_void_p), ("cluster_of_chunk", C.c_void_p),
        ("L", C.c_uint32),
        ("fine_centroid", C.c_void_p), ("fine_radius", C.c_void_p),
        ("fine_token_count", C.c_void_p), ("fine_parent", C.c_void_p),
        ("fine_member_count", C.c_void_p),
        ("P", C.c_uint32),
        ("coarse_centroid", C.c_void_p), ("coarse_radius", C.c_void_p),
        ("coarse_member_off", C.c_void_p), ("coarse_members", C.c_void_p),
        ("structure_aware", C.c_uint32), ("graft_full", C.c_uint32),
    ]


class LcoBudgets(C.Structure):
    _fields_ = [("unit_topk", C.c_uint32), ("mode", C.c_uint32), ("cluster_topk", C.c_uint32),
                ("token_budget", C.c_uint64), ("sink_size", C.c_uint32)]


class LcoResult(C.Structure):
    _fields_ = [("units", C.c_void_p), ("n_units", C.c_uint64),
                ("clusters", C.c_void_p), ("n_clusters", C.c_uint64),
                ("active", C.c_void_p), ("n_active", C.c_uint64),
                ("output", C.c_void_p), ("scanned", C.c_uint64), ("degenerate", C.c_int)]


class LcoGraft(C.Structure):
    _fields_ = [("chunk_id", C.c_uint32), ("cluster_id", C.c_uint32), ("unit_id", C.c_uint32),
                ("centroid_delta", C.c_double), ("fine_radius", C.c_double),
                ("coarse_radius", C.c_double), ("distance_comps", C.c_uint64)]


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"C oracle not built: {LIB_PATH} (run make -C oracle oracle)")
        L = C.CDLL(LIB_PATH)
        L.lco_retrieve.argtypes = [C.POINTER(LcoIndex), C.c_void_p, C.POINTER(LcoBudgets),
                                   C.c_void_p, C.c_size_t, C.c_int, C.POINTER(LcoResult)]
        L.lco_decode_step.argtypes = [C.POINTER(LcoIndex), C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_uint8, C.POINTER(LcoBudgets), C.POINTER(LcoResult),
                                      C.POINTER(C.c_int), C.POINTER(LcoGraft)]
        L.lco_segment_codes.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        L.lco_segment_codes.restype = C.c_size_t
        L.lco_chunk_representative.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_int,
                                               C.c_void_p]
        L.lco_attention.argtypes = [C.c_void_p] * 4 + [C.c_size_t, C.c_size_t, C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data


def segment(codes):
    codes = np.ascontiguousarray(codes, np.uint8)
    out = np.zeros((len(codes) + 1, 4), np.uint32)
    n = lib().lco_segment_codes(_p(codes), len(codes), _p(out))
    return out[:n].copy()


def chunk_representative(keys, pooling=0):
    keys = np.ascontiguousarray(keys, np.float32)
    out = np.empty(keys.shape[1], np.float32)
    rc = lib().lco_chunk_representative(_p(keys), keys.shape[0], keys.shape[1], pooling, _p(out))
    if rc:
        raise ValueError("chunk_representative failed")
    return out


class OracleIndex:
    """Mutable restatement state: TokenStore + HierarchicalIndex + stream cursor."""

    def __init__(self, keys, values, text_code, exp, extra_tokens=0, extra_chunks=0,
                 structure_aware=True, graft_full=False):
        keys = np.asarray(keys, np.float32)
        n, d = keys.shape
        cap = n + extra_tokens
        self.keys = np.zeros((cap, d), np.float32)
        self.keys[:n] = keys
        self.values = np.zeros((cap, d), np.float32)
        self.values[:n] = values
        self.text_code = np.zeros(cap, np.uint8)
        if text_code is not None:
            self.text_code[:n] = text_code
        m = exp.chunk_span.shape[0]
        mcap = m + extra_chunks + 1
        self.chunk_start = np.zeros(mcap, np.uint32)
        self.chunk_end = np.zeros(mcap, np.uint32)
        self.chunk_kind = np.zeros(mcap, np.uint32)
        self.chunk_level = np.zeros(mcap, np.uint32)
        self.chunk_start[:m] = exp.chunk_span[:, 0]
        self.chunk_end[:m] = exp.chunk_span[:, 1]
        self.chunk_kind[:m] = exp.chunk_span[:, 2]
        self.chunk_level[:m] = exp.chunk_span[:, 3]
        self.chunk_rep = np.zeros((mcap, d), np.float32)
        self.chunk_rep[:m] = exp.chunk_rep
        self.cluster_of_chunk = np.zeros(mcap, np.uint32)
        self.cluster_of_chunk[:m] = exp.cluster_of_chunk
        self.fine_centroid = np.ascontiguousarray(exp.fine_centroid, np.float32).copy()
        self.fine_radius = np.ascontiguousarray(exp.fine_radius, np.float64).copy()
        self.fine_token_count = np.ascontiguousarray(exp.fine_token_count, np.uint64).copy()
        self.fine_parent = np.ascontiguousarray(exp.fine_parent, np.uint32).copy()
        self.fine_member_count = np.diff(exp.fine_member_off.astype(np.int64)).astype(np.uint32)
        self.coarse_centroid = np.ascontiguousarray(exp.coarse_centroid, np.float32).copy()
        self.coarse_radius = np.ascontiguousarray(exp.coarse_radius, np.float64).copy()
        self.coarse_member_off = np.ascontiguousarray(exp.coarse_member_off, np.uint32).copy()
        self.coarse_members = np.ascontiguousarray(exp.coarse_members, np.uint32).copy()
        chunked_end = int(exp.chunk_span[-1, 1]) if m else 0
        self.s = LcoIndex(
            d, n, cap, chunked_end, _p(self.keys), _p(self.values), _p(self.text_code),
            m, mcap, _p(self.chunk_start), _p(self.chunk_end), _p(self.chunk_kind),
            _p(self.chunk_level), _p(self.chunk_rep), _p(self.cluster_of_chunk),
            exp.fine_centroid.shape[0], _p(self.fine_centroid), _p(self.fine_radius),
            _p(self.fine_token_count), _p(self.fine_parent), _p(self.fine_member_count),
            exp.coarse_centroid.shape[0], _p(self.coarse_centroid), _p(self.coarse_radius),
            _p(self.coarse_member_off), _p(self.coarse_members), int(structure_aware),
            int(graft_full))
        self.d = d

    @property
    def n_tokens(self):
        return self.s.n_tokens

    def _result(self, n_extra):
        units = np.zeros(max(self.s.P, 1), np.uint32)
        clusters = np.zeros(max(self.s.L, 1), np.uint32)
        active = np.zeros(self.s.n_tokens + n_extra + 1, np.uint32)
        out = np.zeros(self.d, np.float32)
        r = LcoResult(_p(units), 0, _p(clusters), 0, _p(active), 0, _p(out), 0, 0)
        return r, (units, clusters, active, out)

    @staticmethod
    def _pack(r, bufs):
        units, clusters, active, out = bufs
        return dict(units=units[: r.n_units].copy(), clusters=clusters[: r.n_clusters].copy(),
                    active=active[: r.n_active].copy(), output=out.copy(),
                    scanned=int(r.scanned), degenerate=bool(r.degenerate))

    def retrieve(self, q, unit_topk=8, mode=1, cluster_topk=8, token_budget=1024, sink=16,
                 buffer=None, with_output=True):
        q = np.ascontiguousarray(q, np.float32)
        buf = np.ascontiguousarray(buffer if buffer is not None else [], np.uint32)
        b = LcoBudgets(unit_topk, mode, cluster_topk, token_budget, sink)
        r, bufs = self._result(len(buf))
        rc = lib().lco_retrieve(C.byref(self.s), _p(q), C.byref(b), _p(buf) if len(buf) else None,
                                len(buf), int(with_output), C.byref(r))
        if rc:
            raise ValueError(f"lco_retrieve rc={rc}")
        return self._pack(r, bufs)

    def decode_step(self, q, key, value, text_code=0, unit_topk=8, mode=1, cluster_topk=8,
                    token_budget=1024, sink=16):
        q = np.ascontiguousarray(q, np.float32)
        key = np.ascontiguousarray(key, np.float32)
        value = np.ascontiguousarray(value, np.float32)
        b = LcoBudgets(unit_topk, mode, cluster_topk, token_budget, sink)
        r, bufs = self._result(32)
        g = C.c_int(0)
        rep = LcoGraft()
        rc = lib().lco_decode_step(C.byref(self.s), _p(q), _p(key), _p(value), text_code,
                                   C.byref(b), C.byref(r), C.byref(g), C.byref(rep))
        if rc:
            raise ValueError(f"lco_decode_step rc={rc}")
        res = self._pack(r, bufs)
        res["graft"] = None
        if g.value:
            res["graft"] = dict(chunk_id=rep.chunk_id, cluster_id=rep.cluster_id,
                                unit_id=rep.unit_id, distance_comps=int(rep.distance_comps),
                                centroid_delta=rep.centroid_delta, fine_radius=rep.fine_radius,
                                coarse_radius=rep.coarse_radius)
        return res
