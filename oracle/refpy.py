"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/_ref/libtierkv_ref.so`` -- the UNMODIFIED
reference library (``/root/reference/proj/src``) plus ``ref_shim.cpp``.
Used only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs, always as the checker or the timed
reference, never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtierkv_ref.so")

_lib = None

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
vp = C.c_void_p


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        L.tkr_last_error.restype = C.c_char_p
        L.tkr_workload_new.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                       C.c_uint64, C.c_double, C.c_uint64, C.POINTER(vp)]
        L.tkr_workload_free.argtypes = [vp]
        L.tkr_workload_export.argtypes = [vp] + [vp] * 6
        L.tkr_local_queries.argtypes = [C.c_uint64] * 3 + [C.c_double] + [C.c_uint64] * 4 + [f32p]
        L.tkr_rng_draws.argtypes = [C.c_uint64, C.c_uint64, u64p, C.c_uint64, f64p]
        L.tkr_segment.argtypes = [u8p, C.c_uint64, u32p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.tkr_engine_new.argtypes = [f32p, f32p, vp, C.c_uint64, C.c_uint64, vp, C.c_uint64,
                                     C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(vp)]
        L.tkr_engine_free.argtypes = [vp]
        L.tkr_engine_dims.argtypes = [vp, u64p]
        L.tkr_engine_export.argtypes = [vp] + [vp] * 13
        L.tkr_engine_index_bytes.argtypes = [vp, vp, C.c_uint64]
        L.tkr_engine_index_bytes.restype = C.c_uint64
        L.tkr_engine_store_export.argtypes = [vp, vp, vp]
        L.tkr_save_index.argtypes = [vp, C.c_char_p]
        L.tkr_engine_load.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.POINTER(vp)]
        L.tkr_oracle_topk.argtypes = [vp, f32p, C.c_uint64, C.c_uint64, u32p, C.c_uint64,
                                      C.POINTER(C.c_uint64)]
        L.tkr_retrieve.argtypes = [vp, f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint64, C.c_uint32, vp, C.c_uint64, C.c_int,
                                   u32p, C.c_uint64, u32p, C.c_uint64, u32p, C.c_uint64,
                                   f32p, u64p]
        L.tkr_sparse_attention.argtypes = [vp, f32p, C.c_uint64, u32p, C.c_uint64, f32p]
        L.tkr_full_attention.argtypes = [vp, f32p, C.c_uint64, f32p]
        L.tkr_decode_step.argtypes = [vp, f32p, f32p, f32p, C.c_uint8, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_uint64, C.c_uint32,
                                      u32p, C.c_uint64, u32p, C.c_uint64, u32p, C.c_uint64,
                                      f32p, u64p, f64p, u64p, f64p]
        L.tkr_push_and_graft.argtypes = [vp, f32p, f32p, C.c_uint8, u64p, f64p]
        L.tkr_chunk_representative.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint32, f32p]
        L.tkr_audit.argtypes = [vp, f32p, C.c_uint64, C.c_double]
        L.tkr_audit.restype = C.c_uint64
        L.tkr_time_retrieve.argtypes = [C.POINTER(vp), C.c_uint64, f32p, C.c_uint64, C.c_uint64,
                                        C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int,
                                        C.c_int, C.POINTER(C.c_uint64)]
        L.tkr_time_retrieve.restype = C.c_double
        L.tkr_threads.restype = C.c_int
        L.tkr_set_thread_team.argtypes = [C.c_int]
        _lib = L
    return _lib


class RefError(Exception):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().tkr_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(msg)
    raise RefError(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class Workload:
    keys: np.ndarray      # [n, d] f32
    values: np.ndarray    # [n, d] f32
    text_code: np.ndarray  # [n] u8: 0 "", 1 "\n", 2 "}"
    queries: np.ndarray   # [qc, d] f32
    centers: np.ndarray   # [n_blobs, d]
    token_blob: np.ndarray


def gen_workload(n_tokens, d=128, seed=1, n_blobs=8, concentration=3.0, query_count=4,
                 locality=0.8) -> Workload:
    """gen_clustered_workload (workload.cpp:110-169)."""
    h = vp()
    _check(lib().tkr_workload_new(n_tokens, d, n_blobs, concentration, query_count, locality,
                                  seed, C.byref(h)))
    try:
        keys = np.empty((n_tokens, d), np.float32)
        values = np.empty((n_tokens, d), np.float32)
        tc = np.empty(n_tokens, np.uint8)
        qs = np.empty((query_count, d), np.float32)
        cs = np.empty((n_blobs, d), np.float32)
        tb = np.empty(n_tokens, np.uint32)
        lib().tkr_workload_export(h, _ptr(keys), _ptr(values), _ptr(tc), _ptr(qs), _ptr(cs),
                                  _ptr(tb))
    finally:
        lib().tkr_workload_free(h)
    return Workload(keys, values, tc, qs, cs, tb)


def local_queries(n_tokens, d, n_blobs, conc, seed, blob, count, qseed):
    out = np.empty((count, d), np.float32)
    _check(lib().tkr_local_queries(n_tokens, d, n_blobs, conc, seed, blob, count, qseed, out))
    return out


def segment(text_code: np.ndarray) -> np.ndarray:
    """chunker segment() with ChunkPolicy::defaults() -> [n_spans, 4] (start,end,kind,level)."""
    tc = np.ascontiguousarray(text_code, np.uint8)
    cap = len(tc) + 1
    out = np.empty((cap, 4), np.uint32)
    n = C.c_uint64()
    _check(lib().tkr_segment(tc, len(tc), out, cap, C.byref(n)))
    return out[: n.value].copy()


@dataclass
class IndexExport:
    dim: int
    chunk_span: np.ndarray       # [M,4]
    chunk_rep: np.ndarray        # [M,d]
    fine_centroid: np.ndarray    # [L,d]
    fine_radius: np.ndarray      # [L] f64
    fine_token_count: np.ndarray  # [L] u64
    fine_parent: np.ndarray      # [L]
    fine_member_off: np.ndarray  # [L+1]
    fine_members: np.ndarray
    coarse_centroid: np.ndarray  # [P,d]
    coarse_radius: np.ndarray    # [P]
    coarse_member_off: np.ndarray
    coarse_members: np.ndarray
    cluster_of_chunk: np.ndarray

    @property
    def n_chunks(self):
        return self.chunk_span.shape[0]

    @property
    def n_clusters(self):
        return self.fine_centroid.shape[0]

    @property
    def n_units(self):
        return self.coarse_centroid.shape[0]


class RefEngine:
    """The reference StreamState (store + HierarchicalIndex) built by build_index."""

    def __init__(self, keys, values, text_code=None, spans=None, avg_chunks=2.0, max_units=64,
                 iters=10, pooling=0, seed=0, structure_aware=True, graft_full=False, _handle=None):
        if _handle is not None:  # RefEngine.load
            self.h = _handle
            self.d = self.dims()[0]
            return
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        n, d = keys.shape
        self.d = d
        tc = None if text_code is None else np.ascontiguousarray(text_code, np.uint8)
        sp = None if spans is None else np.ascontiguousarray(spans, np.uint32)
        self.h = vp()
        _check(lib().tkr_engine_new(keys, values, _ptr(tc), n, d, _ptr(sp),
                                    0 if sp is None else sp.shape[0], avg_chunks, max_units,
                                    iters, pooling, seed, int(structure_aware), int(graft_full),
                                    C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().tkr_engine_free(self.h)
            self.h = None

    @classmethod
    def load(cls, path, structure_aware=True, graft_full=False) -> "RefEngine":
        """StreamState over the reference's load_index (serialize.cpp:150-220)."""
        h = vp()
        _check(lib().tkr_engine_load(path.encode(), int(structure_aware), int(graft_full), C.byref(h)))
        return cls(None, None, _handle=h)

    def save(self, path):
        """The reference's save_index (serialize.cpp:127-148)."""
        _check(lib().tkr_save_index(self.h, path.encode()))

    def oracle_topk(self, q, budget):
        """eval::oracle_topk_tokens (evaluator.cpp:43-64)."""
        q = np.ascontiguousarray(q, np.float32)
        n = self.dims()[4]
        out = np.empty(max(n, 1), np.uint32)
        k = C.c_uint64()
        _check(lib().tkr_oracle_topk(self.h, q, len(q), budget, out, len(out), C.byref(k)))
        return out[: k.value].copy()

    def dims(self):
        out = np.zeros(8, np.uint64)
        lib().tkr_engine_dims(self.h, out)
        return [int(x) for x in out]

    def export(self) -> IndexExport:
        d, m, l, p, _, fm, cm, _ = self.dims()
        e = IndexExport(
            d, np.empty((m, 4), np.uint32), np.empty((m, d), np.float32),
            np.empty((l, d), np.float32), np.empty(l, np.float64), np.empty(l, np.uint64),
            np.empty(l, np.uint32), np.empty(l + 1, np.uint32), np.empty(fm, np.uint32),
            np.empty((p, d), np.float32), np.empty(p, np.float64), np.empty(p + 1, np.uint32),
            np.empty(cm, np.uint32), np.empty(m, np.uint32))
        lib().tkr_engine_export(self.h, *[_ptr(a) for a in (
            e.chunk_span, e.chunk_rep, e.fine_centroid, e.fine_radius, e.fine_token_count,
            e.fine_parent, e.fine_member_off, e.fine_members, e.coarse_centroid,
            e.coarse_radius, e.coarse_member_off, e.coarse_members, e.cluster_of_chunk)])
        return e

    def index_bytes(self) -> bytes:
        n = lib().tkr_engine_index_bytes(self.h, None, 0)
        buf = np.empty(n, np.uint8)
        lib().tkr_engine_index_bytes(self.h, _ptr(buf), n)
        return buf.tobytes()

    def store(self):
        n = self.dims()[4]
        k = np.empty((n, self.d), np.float32)
        v = np.empty((n, self.d), np.float32)
        lib().tkr_engine_store_export(self.h, _ptr(k), _ptr(v))
        return k, v

    def retrieve(self, q, unit_topk=8, mode=1, cluster_topk=8, token_budget=1024, sink=16,
                 buffer=None, with_output=True):
        q = np.ascontiguousarray(q, np.float32)
        d, m, l, p, n, _, _, _ = self.dims()
        buf = None if buffer is None else np.ascontiguousarray(buffer, np.uint32)
        units = np.empty(max(p, 1), np.uint32)
        clusters = np.empty(max(l, 1), np.uint32)
        active = np.empty(max(n + (0 if buf is None else len(buf)), 1), np.uint32)
        out = np.zeros(d, np.float32)
        counts = np.zeros(5, np.uint64)
        _check(lib().tkr_retrieve(self.h, q, len(q), unit_topk, mode, cluster_topk, token_budget,
                                  sink, _ptr(buf), 0 if buf is None else len(buf),
                                  int(with_output), units, len(units), clusters, len(clusters),
                                  active, len(active), out, counts))
        return dict(units=units[: counts[0]].copy(), clusters=clusters[: counts[1]].copy(),
                    active=active[: counts[2]].copy(), output=out if with_output else None,
                    scanned=int(counts[3]), degenerate=bool(counts[4]))

    def sparse_attention(self, q, ids):
        q = np.ascontiguousarray(q, np.float32)
        ids = np.ascontiguousarray(ids, np.uint32)
        out = np.zeros(len(q), np.float32)
        _check(lib().tkr_sparse_attention(self.h, q, len(q), ids, len(ids), out))
        return out

    def full_attention(self, q):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(len(q), np.float32)
        _check(lib().tkr_full_attention(self.h, q, len(q), out))
        return out

    def decode_step(self, q, key, value, text_code=0, unit_topk=8, mode=1, cluster_topk=8,
                    token_budget=1024, sink=16):
        q = np.ascontiguousarray(q, np.float32)
        key = np.ascontiguousarray(key, np.float32)
        value = np.ascontiguousarray(value, np.float32)
        d, m, l, p, n, _, _, _ = self.dims()
        units = np.empty(max(p, 1), np.uint32)
        clusters = np.empty(max(l, 1), np.uint32)
        active = np.empty(n + 1, np.uint32)
        out = np.zeros(d, np.float32)
        counts = np.zeros(5, np.uint64)
        stab = np.zeros(2, np.float64)
        gu = np.zeros(8, np.uint64)
        gf = np.zeros(3, np.float64)
        _check(lib().tkr_decode_step(self.h, q, key, value, text_code, unit_topk, mode,
                                     cluster_topk, token_budget, sink, units, len(units),
                                     clusters, len(clusters), active, len(active), out, counts,
                                     stab, gu, gf))
        res = dict(units=units[: counts[0]].copy(), clusters=clusters[: counts[1]].copy(),
                   active=active[: counts[2]].copy(), output=out, scanned=int(counts[3]),
                   degenerate=bool(counts[4]), jaccard=float(stab[0]), window_hit=float(stab[1]))
        res["graft"] = None
        if gu[0]:
            res["graft"] = dict(chunk_id=int(gu[1]), cluster_id=int(gu[2]), unit_id=int(gu[3]),
                                distance_comps=int(gu[4]), span=(int(gu[5]), int(gu[6])),
                                centroid_delta=float(gf[0]), fine_radius=float(gf[1]),
                                coarse_radius=float(gf[2]))
        return res

    def push_and_graft(self, key, value, text_code=0):
        key = np.ascontiguousarray(key, np.float32)
        value = np.ascontiguousarray(value, np.float32)
        gu = np.zeros(8, np.uint64)
        gf = np.zeros(3, np.float64)
        _check(lib().tkr_push_and_graft(self.h, key, value, text_code, gu, gf))
        if not gu[0]:
            return None
        return dict(chunk_id=int(gu[1]), cluster_id=int(gu[2]), unit_id=int(gu[3]),
                    distance_comps=int(gu[4]), centroid_delta=float(gf[0]),
                    fine_radius=float(gf[1]), coarse_radius=float(gf[2]))

    def audit(self, queries, tol=1e-6):
        q = np.ascontiguousarray(queries, np.float32)
        return int(lib().tkr_audit(self.h, q, q.shape[0], tol))


def chunk_representative(keys, pooling=0):
    keys = np.ascontiguousarray(keys, np.float32)
    out = np.empty(keys.shape[1], np.float32)
    _check(lib().tkr_chunk_representative(keys, keys.shape[0], keys.shape[1], pooling, out))
    return out


def rng_draws(seed, n_u64, n_gauss):
    a = np.empty(max(n_u64, 1), np.uint64)
    b = np.empty(max(n_gauss, 1), np.float64)
    lib().tkr_rng_draws(seed, n_u64, a, n_gauss, b)
    return a[:n_u64], b[:n_gauss]


def time_retrieve(engines, queries, token_budget=2048, unit_topk=8, sink=16, reps=1, mode=1,
                  threads=0):
    """Wall seconds for reps x (every engine x its queries) reference retrieve() calls."""
    arr = (vp * len(engines))(*[e.h for e in engines])
    q = np.ascontiguousarray(queries, np.float32)
    nq_per = q.shape[0] // len(engines)
    chk = C.c_uint64()
    secs = lib().tkr_time_retrieve(arr, len(engines), q, nq_per, q.shape[1], unit_topk,
                                   token_budget, sink, reps, mode, threads, C.byref(chk))
    return secs, chk.value


def set_thread_team(n):
    """OpenMP team size of parallel regions the calling thread starts."""
    lib().tkr_set_thread_team(int(n))


def threads():
    return lib().tkr_threads()


def fnv1a64(buf: bytes) -> int:
    """FNV-1a-64 (offset basis 1469598103934665603, prime 1099511628211) via the C oracle."""
    from . import cpy
    L = cpy.lib()
    L.lco_fnv1a64.restype = C.c_uint64
    L.lco_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
    return int(L.lco_fnv1a64(buf, len(buf)))
