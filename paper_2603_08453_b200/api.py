"""Host-side mirror of the reference's index/decode interface over the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/tierkv/{retriever,streamer,index}.hpp):

* ``Budgets`` / ``SelectionMode``       -- retriever.hpp:11-21
* ``RetrievalResult``                   -- retriever.hpp:23-30
* ``retrieve`` / ``retrieve_ids`` / ``sparse_attention`` -- retriever.hpp:34-58
* ``GraftReport`` / ``DecodeOutcome`` / ``StreamState`` -- streamer.hpp:27-85

The compute runs in ``liblychee_b200.so`` (sm_100a); torch is only used to
hold device buffers.  ``Engine`` is the batched form: many (layer, KV head,
sequence) slots per GPU and ``group`` query heads per slot.
"""
from __future__ import annotations

import ctypes as C
import enum
from collections import deque
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

try:  # plumbing only: device buffers and streams
    import torch
except Exception:  # pragma: no cover
    torch = None


class SelectionMode(enum.IntEnum):
    fixed_cluster_count = 0
    token_budget = 1


class GraftSearch(enum.IntEnum):
    scoped = 0
    full = 1


@dataclass
class Budgets:
    """tierkv::Budgets (retriever.hpp:13-21)."""
    unit_topk: int = 8
    mode: SelectionMode = SelectionMode.token_budget
    cluster_topk: int = 8
    token_budget: int = 1024
    sink_size: int = 16

    def validate(self):
        # Budgets::validate (retriever.cpp:11-17)
        if self.unit_topk < 1:
            raise ValueError("unit_topk must be >= 1")
        if self.mode == SelectionMode.fixed_cluster_count and self.cluster_topk < 1:
            raise ValueError("cluster_topk must be >= 1")
        if self.mode == SelectionMode.token_budget and self.token_budget < 1:
            raise ValueError("token_budget must be >= 1")

    def c(self):
        return L.Budgets_(self.unit_topk, int(self.mode), self.cluster_topk, self.token_budget,
                          self.sink_size)


@dataclass
class RetrievalResult:
    """tierkv::RetrievalResult (retriever.hpp:23-30)."""
    selected_units: np.ndarray
    selected_clusters: np.ndarray
    active_token_ids: np.ndarray
    output: Optional[np.ndarray]
    scanned_centroids: int
    degenerate: bool


@dataclass
class GraftReport:
    """tierkv::GraftReport (streamer.hpp:27-35)."""
    chunk_id: int
    cluster_id: int
    unit_id: int
    centroid_delta: float
    fine_radius: float
    coarse_radius: float
    distance_comps: int


@dataclass
class DecodeOutcome:
    """tierkv::DecodeOutcome (streamer.hpp:37-42)."""
    retrieval: RetrievalResult
    jaccard: float = 0.0
    window_hit: float = 0.0
    graft: Optional[GraftReport] = None


@dataclass
class IndexConfig:
    """tierkv::IndexConfig (index.hpp:13-22) as index_to_bytes serializes it."""
    avg_chunks_per_cluster: float = 2.0
    max_coarse_units: int = 64
    kmeans_iters: int = 10
    pooling: int = 0
    elem_bytes: int = 2
    seed: int = 0

    def c(self):
        return L.IndexConfig_(self.avg_chunks_per_cluster, self.max_coarse_units, self.kmeans_iters,
                              self.pooling, self.elem_bytes, self.seed)

    @classmethod
    def from_c(cls, c):
        return cls(c.avg_chunks_per_cluster, c.max_coarse_units, c.kmeans_iters, c.pooling,
                   c.elem_bytes, c.seed)


@dataclass
class HostIndex:
    """tierkv::HierarchicalIndex in SoA form, reference numbering (index.hpp:25-73)."""
    dim: int
    chunk_span: np.ndarray        # [M,4] u32 start, end, kind, level
    chunk_rep: np.ndarray         # [M,d] f32
    fine_centroid: np.ndarray     # [L,d] f32
    fine_radius: np.ndarray       # [L] f64
    fine_token_count: np.ndarray  # [L] u64
    fine_parent: np.ndarray       # [L] u32
    fine_member_off: np.ndarray   # [L+1] u32
    fine_members: np.ndarray      # u32
    coarse_centroid: np.ndarray   # [P,d] f32
    coarse_radius: np.ndarray     # [P] f64
    coarse_member_off: np.ndarray  # [P+1] u32
    coarse_members: np.ndarray    # u32
    cluster_of_chunk: np.ndarray  # [M] u32

    @property
    def n_chunks(self):
        return int(self.chunk_span.shape[0])

    @property
    def n_clusters(self):
        return int(self.fine_centroid.shape[0])

    @property
    def n_units(self):
        return int(self.coarse_centroid.shape[0])

    @classmethod
    def from_export(cls, e) -> "HostIndex":
        return cls(e.dim, *[np.ascontiguousarray(getattr(e, f)) for f in (
            "chunk_span", "chunk_rep", "fine_centroid", "fine_radius", "fine_token_count",
            "fine_parent", "fine_member_off", "fine_members", "coarse_centroid", "coarse_radius",
            "coarse_member_off", "coarse_members", "cluster_of_chunk")])

    def _c(self):
        arrs = dict(
            chunk_span=np.ascontiguousarray(self.chunk_span, np.uint32),
            chunk_rep=None if self.chunk_rep is None else np.ascontiguousarray(self.chunk_rep, np.float32),
            fine_centroid=np.ascontiguousarray(self.fine_centroid, np.float32),
            fine_radius=np.ascontiguousarray(self.fine_radius, np.float64),
            fine_token_count=np.ascontiguousarray(self.fine_token_count, np.uint64),
            fine_parent=np.ascontiguousarray(self.fine_parent, np.uint32),
            fine_member_off=np.ascontiguousarray(self.fine_member_off, np.uint32),
            fine_members=np.ascontiguousarray(self.fine_members, np.uint32),
            coarse_centroid=np.ascontiguousarray(self.coarse_centroid, np.float32),
            coarse_radius=np.ascontiguousarray(self.coarse_radius, np.float64),
            coarse_member_off=np.ascontiguousarray(self.coarse_member_off, np.uint32),
            coarse_members=np.ascontiguousarray(self.coarse_members, np.uint32),
            cluster_of_chunk=np.ascontiguousarray(self.cluster_of_chunk, np.uint32))
        s = L.HostIndex_(self.dim, self.n_chunks, self.n_clusters, self.n_units,
                         *[None if arrs[k] is None else arrs[k].ctypes.data for k in (
                             "chunk_span", "chunk_rep", "fine_centroid", "fine_radius",
                             "fine_token_count", "fine_parent", "fine_member_off", "fine_members",
                             "coarse_centroid", "coarse_radius", "coarse_member_off",
                             "coarse_members", "cluster_of_chunk")])
        return s, arrs  # keep arrays alive while the struct is used

    @classmethod
    def empty(cls, dims) -> "HostIndex":
        d, m, l, p, _, fm, cm, _ = [int(x) for x in dims]
        return cls(d, np.zeros((m, 4), np.uint32), np.zeros((m, d), np.float32),
                   np.zeros((l, d), np.float32), np.zeros(l, np.float64), np.zeros(l, np.uint64),
                   np.zeros(l, np.uint32), np.zeros(l + 1, np.uint32), np.zeros(max(fm, 1), np.uint32),
                   np.zeros((p, d), np.float32), np.zeros(p, np.float64), np.zeros(p + 1, np.uint32),
                   np.zeros(max(cm, 1), np.uint32), np.zeros(m, np.uint32))

    def _fill_from(self, keep, fm, cm):
        for k, v in keep.items():
            if v is not None:
                setattr(self, k, v)
        self.fine_members = self.fine_members[:fm]
        self.coarse_members = self.coarse_members[:cm]
        return self


# ---- TKIX codec (serialize.cpp:88-220), host only ----------------------------
def index_to_bytes(ix: HostIndex, cfg: Optional[IndexConfig] = None) -> bytes:
    """index_to_bytes (serialize.cpp:88-125) of a host index."""
    s, keep = ix._c()
    c = (cfg or IndexConfig()).c()
    n = L.u64()
    L.check(L.lib().lc_tkix_encode(C.byref(s), C.byref(c), None, 0, C.byref(n)))
    buf = np.zeros(n.value, np.uint8)
    L.check(L.lib().lc_tkix_encode(C.byref(s), C.byref(c), buf.ctypes.data, n.value, C.byref(n)))
    return buf.tobytes()


def index_from_bytes(data: bytes):
    """The index part of load_index (serialize.cpp:150-208) -> (HostIndex, IndexConfig)."""
    buf = np.frombuffer(data, np.uint8).copy()
    dims = np.zeros(8, np.uint64)
    L.check(L.lib().lc_tkix_decode_dims(buf.ctypes.data, len(buf), dims.ctypes.data))
    ix = HostIndex.empty(dims)
    s, keep = ix._c()
    c = L.IndexConfig_()
    L.check(L.lib().lc_tkix_decode(buf.ctypes.data, len(buf), C.byref(s), C.byref(c)))
    return ix._fill_from(keep, int(dims[5]), int(dims[6])), IndexConfig.from_c(c)


# ---- bf16 helpers (the device KV cache is bf16) ------------------------------
def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest even (as torch / cuda_bf16)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    nan = np.isnan(np.asarray(x, np.float32))
    out = rounded.astype(np.uint16)
    out[nan] = 0x7FC0
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 values rounded to bf16 and widened back (what the device stores)."""
    return (bf16_bits(x).astype(np.uint32) << 16).view(np.float32)


_REPORT_DT = np.dtype([("chunk_id", "<u4"), ("cluster_id", "<u4"), ("unit_id", "<u4"),
                       ("_pad", "<u4"), ("centroid_delta", "<f8"), ("fine_radius", "<f8"),
                       ("coarse_radius", "<f8"), ("distance_comps", "<u8")])


def _ptr(t):
    if t is None:
        return None
    if torch is not None and isinstance(t, torch.Tensor):
        return t.data_ptr()
    return t.ctypes.data


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None) if torch is not None else None


def _stream_ptr(stream):
    if stream is None:
        if torch is not None and torch.cuda.is_available():
            if _raw_stream is not None:  # the current stream's handle without a Stream object (hot loops)
                return _raw_stream(torch.cuda.current_device())
            return torch.cuda.current_stream().cuda_stream
        return None
    return getattr(stream, "cuda_stream", stream)


class Engine:
    """All slots resident on one GPU (lc_index_t)."""

    def __init__(self, n_slots: int, dim: int = 128, group: int = 4, cap_tokens: int = 1 << 16,
                 cap_chunks: int = 1 << 13, cap_clusters: int = 1 << 12, cap_units: int = 64,
                 structure_aware: bool = True, graft_full: bool = False,
                 keep_reps: bool = True, pooling: int = 0, device: int = 0, max_candidates: int = 0,
                 slot_groups: int = 0, kv_f32: bool = False):
        """kv_f32: keep K/V in fp32 exactly as given, attention in fp64 (the
        reference-exact mode; head dims 8/16/32 also allowed for group 1 or 4)."""
        self.desc = L.IndexDesc(n_slots, dim, group, cap_tokens, cap_chunks, cap_clusters,
                                cap_units, max_candidates, int(structure_aware),
                                int(graft_full), int(keep_reps), pooling, slot_groups, device, int(kv_f32))
        self.kv_f32 = bool(kv_f32)
        self.h = C.c_void_p()
        L.check(L.lib().lc_index_create(C.byref(self.desc), C.byref(self.h)))
        got = L.IndexDesc()
        L.check(L.lib().lc_index_get_desc(self.h, C.byref(got)))
        self.desc = got
        self.n_slots, self.dim, self.group = n_slots, dim, group
        self.device = device
        self._reports = None

    def close(self):
        if getattr(self, "h", None):
            L.lib().lc_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- slots ----
    def _kv(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x)
        if self.kv_f32:
            return np.ascontiguousarray(x, np.float32)
        return np.ascontiguousarray(x if x.dtype == np.uint16 else bf16_bits(x))

    def upload_slot(self, slot: int, ix: HostIndex, keys: np.ndarray, values: np.ndarray):
        kb = self._kv(keys)
        vb = self._kv(values)
        kb = np.ascontiguousarray(kb)
        vb = np.ascontiguousarray(vb)
        s, keep = ix._c()
        L.check(L.lib().lc_index_upload_slot(self.h, slot, C.byref(s), kb.ctypes.data,
                                             vb.ctypes.data, kb.shape[0]))

    def kv_upload(self, slot: int, keys: np.ndarray, values: np.ndarray):
        kb = self._kv(keys)
        vb = self._kv(values)
        L.check(L.lib().lc_kv_upload_slot(self.h, slot, kb.ctypes.data, vb.ctypes.data, kb.shape[0]))

    def kv_download(self, slot: int, n: int):
        dt = np.float32 if self.kv_f32 else np.uint16
        k = np.zeros((n, self.dim), dt)
        v = np.zeros((n, self.dim), dt)
        L.check(L.lib().lc_kv_download_slot(self.h, slot, k.ctypes.data, v.ctypes.data, n))
        return k, v

    def gen_workload(self, n_tokens: int, seeds, n_blobs=8, concentration=3.0, query_count=4,
                     query_locality=0.8):
        """gen_clustered_workload token streams written straight into every slot
        (GPU); returns (text codes [S, n], queries [S, query_count, d])."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        codes = np.zeros((self.n_slots, n_tokens), np.uint8)
        qs = np.zeros((self.n_slots, query_count, self.dim), np.float32)
        L.check(L.lib().lc_gen_workload(self.h, n_tokens, n_blobs, concentration, query_count,
                                        query_locality, seeds.ctypes.data, codes.ctypes.data,
                                        qs.ctypes.data))
        return codes, qs

    def build_index(self, n_tokens, spans_per_slot, seeds, avg_chunks_per_cluster=2.0,
                    max_coarse_units=64, kmeans_iters=10):
        """build_index (index.cpp:155-243) for every slot on the GPU from its resident keys."""
        n_tokens = np.ascontiguousarray(n_tokens, np.uint32)
        spans = np.ascontiguousarray(np.concatenate([np.asarray(s, np.uint32).reshape(-1, 4)
                                                     for s in spans_per_slot]), np.uint32)
        off = np.zeros(self.n_slots + 1, np.uint64)
        off[1:] = np.cumsum([len(s) for s in spans_per_slot])
        seeds = np.ascontiguousarray(seeds, np.uint64)
        L.check(L.lib().lc_index_build(self.h, n_tokens.ctypes.data, spans.ctypes.data, off.ctypes.data,
                                       avg_chunks_per_cluster, max_coarse_units, kmeans_iters,
                                       seeds.ctypes.data))

    def slot_dims(self, slot: int):
        out = np.zeros(8, np.uint64)
        L.check(L.lib().lc_index_slot_dims(self.h, slot, out.ctypes.data))
        return [int(x) for x in out]

    def download_slot(self, slot: int) -> HostIndex:
        dims = self.slot_dims(slot)
        ix = HostIndex.empty(dims)
        s, keep = ix._c()
        L.check(L.lib().lc_index_download_slot(self.h, slot, C.byref(s)))
        return ix._fill_from(keep, dims[5], dims[6])

    # ---- TKIX <-> device (serialize.cpp:88-220) ----
    def set_config(self, slot: int, cfg: IndexConfig):
        c = cfg.c()
        L.check(L.lib().lc_index_set_config(self.h, slot, C.byref(c)))

    def get_config(self, slot: int) -> IndexConfig:
        c = L.IndexConfig_()
        L.check(L.lib().lc_index_get_config(self.h, slot, C.byref(c)))
        return IndexConfig.from_c(c)

    def index_bytes(self, slot: int) -> bytes:
        """index_to_bytes(state.index()) of the slot's live index (grafts included)."""
        n = L.u64()
        L.check(L.lib().lc_index_to_bytes(self.h, slot, None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        L.check(L.lib().lc_index_to_bytes(self.h, slot, buf.ctypes.data, n.value, C.byref(n)))
        return buf.tobytes()

    def save_index(self, slot: int, path: str, texts: Optional[Sequence[str]] = None):
        """save_index (serialize.cpp:127-148): TKIX file with the slot's token store."""
        tb, offs = None, None
        if texts is not None:
            enc = [t.encode() for t in texts]
            offs = np.zeros(len(enc) + 1, np.uint64)
            offs[1:] = np.cumsum([len(e) for e in enc])
            tb = np.frombuffer(b"".join(enc) + b"\0", np.uint8).copy()
        L.check(L.lib().lc_index_save(self.h, slot, path.encode(), _ptr(tb), _ptr(offs)))

    def load_index(self, slot: int, path: str):
        """load_index (serialize.cpp:150-220) into a slot; returns the store's texts."""
        n = L.u64()
        L.check(L.lib().lc_index_load(self.h, slot, path.encode(), None, 0, None, 0, C.byref(n)))
        offs = np.zeros(n.value + 1, np.uint64)
        L.check(L.lib().lc_index_load(self.h, slot, path.encode(), None, 0, offs.ctypes.data, len(offs),
                                      C.byref(n)))
        tb = np.zeros(max(int(offs[-1]), 1), np.uint8)
        L.check(L.lib().lc_index_load(self.h, slot, path.encode(), tb.ctypes.data, len(tb), offs.ctypes.data,
                                      len(offs), C.byref(n)))
        raw = tb.tobytes()
        return [raw[int(offs[i]):int(offs[i + 1])].decode() for i in range(n.value)]

    # ---- decode-step operations ----
    def retrieve(self, q, budgets: Budgets, buffer: str = "none", out=None, buf_off=None,
                 buf_ids=None, stream=None):
        """Batched retrieve() for every (slot, query head); q: cuda f32 [S, G, d]."""
        flags = {"none": L.LC_BUFFER_NONE, "stream": L.LC_BUFFER_STREAM, "list": L.LC_BUFFER_LIST}[buffer]
        b = budgets.c()
        L.check(L.lib().lc_retrieve(self.h, _ptr(q), C.byref(b), flags, _ptr(buf_off),
                                    _ptr(buf_ids), _ptr(out), _stream_ptr(stream)))
        return out

    def retrieve_slots(self, first: int, count: int, q, budgets: Budgets, out=None, buffer: str = "none",
                       stream=None):
        """retrieve() for slots [first, first + count) only (one layer of a
        layer-by-layer decode); q / out keep the engine-wide [S, G, d] layout."""
        flags = {"none": L.LC_BUFFER_NONE, "stream": L.LC_BUFFER_STREAM}[buffer]
        b = self._budgets_c(budgets)
        L.check(L.lib().lc_retrieve_slots(self.h, first, count, _ptr(q), C.byref(b), flags, None, None,
                                          _ptr(out), _stream_ptr(stream)))
        return out

    def set_gather(self, peer_out, peer_flag, row_of_slot, my_flag, rows_per_wait):
        """Fused all-gather epilogue (lc_set_gather): peer_out / peer_flag are
        device pointers (ints) of every rank's gather buffer and arrival
        counter, row_of_slot the gather-buffer row of each of this engine's
        slots, my_flag this rank's counter.  Empty lists turn it off."""
        n = len(peer_out)
        po = np.ascontiguousarray(peer_out, np.uint64)
        pf = np.ascontiguousarray(peer_flag, np.uint64)
        rows = np.ascontiguousarray(row_of_slot, np.uint32)
        L.check(L.lib().lc_set_gather(self.h, n, po.ctypes.data if n else None, pf.ctypes.data if n else None,
                                      rows.ctypes.data if n else None, int(my_flag) if n else 0,
                                      int(rows_per_wait)))

    def gather_wait(self, stream=None):
        L.check(L.lib().lc_gather_wait(self.h, _stream_ptr(stream)))

    def retrieve_host(self, q_host: np.ndarray, budgets: Budgets, out_host: np.ndarray,
                      buffer: str = "none", stream=None):
        """retrieve() for every (slot, head) with q and the outputs in host memory
        (page-locked buffers are read and written in place by the kernels)."""
        flags = L.LC_BUFFER_STREAM if buffer == "stream" else L.LC_BUFFER_NONE
        if buffer not in ("none", "stream"):
            raise ValueError("buffer must be 'none' or 'stream'")
        key = (budgets.unit_topk, int(budgets.mode), budgets.cluster_topk, budgets.token_budget, budgets.sink_size)
        bc = self._host_budgets.get(key) if hasattr(self, "_host_budgets") else None
        if bc is None:  # one ctypes struct per distinct budgets (the call is on the decode hot loop)
            if not hasattr(self, "_host_budgets"):
                self._host_budgets = {}
            bc = self._host_budgets[key] = budgets.c()
        rc = L.lib().lc_retrieve_host(self.h, q_host.ctypes.data, C.byref(bc), flags, out_host.ctypes.data,
                                      _stream_ptr(stream))
        if rc:
            L.check(rc)
        return out_host

    def sparse_attention(self, q, out, stream=None):
        L.check(L.lib().lc_sparse_attention(self.h, _ptr(q), _ptr(out), _stream_ptr(stream)))
        return out

    def selection(self, slot: int, g: int, active: bool = True, output=None, staged: bool = False,
                  stream=None) -> RetrievalResult:
        """staged=True: through lc_selection_stage on `stream` + one stream
        sync + lc_selection_read_staged (the C++ drop-in's path)."""
        d, m, l, p, n, _, _, _ = self.slot_dims(slot)
        info = L.SelectionInfo_()
        units = np.zeros(max(p, 1), np.uint32)
        clusters = np.zeros(max(l, 1), np.uint32)
        act = np.zeros(max(n + 1024, 1), np.uint32) if active else None
        if staged:
            L.check(L.lib().lc_selection_stage(self.h, slot, g, _stream_ptr(stream)))
            (stream or torch.cuda.current_stream()).synchronize()
            L.check(L.lib().lc_selection_read_staged(self.h, C.byref(info), units.ctypes.data, len(units),
                                                     clusters.ctypes.data, len(clusters), _ptr(act),
                                                     0 if act is None else len(act)))
        else:
            L.check(L.lib().lc_selection_download(self.h, slot, g, C.byref(info), units.ctypes.data, len(units),
                                                  clusters.ctypes.data, len(clusters), _ptr(act),
                                                  0 if act is None else len(act)))
        if info.error:
            raise L.LcError(L.LC_ERUNTIME, f"device selection error bits 0x{info.error:x}")
        return RetrievalResult(units[: info.n_units].copy(), clusters[: info.n_clusters].copy(),
                               act[: info.n_active].copy() if active else None, output,
                               int(info.scanned_centroids), bool(info.degenerate))

    def selection_info(self, slot: int, g: int):
        info = L.SelectionInfo_()
        L.check(L.lib().lc_selection_download(self.h, slot, g, C.byref(info), None, 0, None, 0, None, 0))
        return info

    def kv_append(self, keys_bf16, values_bf16, stream=None):
        L.check(L.lib().lc_kv_append(self.h, _ptr(keys_bf16), _ptr(values_bf16), _stream_ptr(stream)))

    def _report_buf(self):
        if self._reports is None:
            self._reports = torch.zeros(self.n_slots * _REPORT_DT.itemsize, dtype=torch.uint8,
                                        device=f"cuda:{self.device}")
        return self._reports

    def graft(self, take: np.ndarray, kind=None, level=None, stream=None):
        take = np.ascontiguousarray(take, np.uint32)
        kind = None if kind is None else np.ascontiguousarray(kind, np.uint32)
        level = None if level is None else np.ascontiguousarray(level, np.uint32)
        rb = self._report_buf()
        L.check(L.lib().lc_graft(self.h, take.ctypes.data, _ptr(kind), _ptr(level), rb.data_ptr(),
                                 _stream_ptr(stream)))
        return rb

    def reports(self) -> np.ndarray:
        return self._report_buf().cpu().numpy().view(_REPORT_DT)

    def decode_step(self, q, keys_bf16, values_bf16, budgets: Budgets, take=None, kind=None,
                    level=None, out=None, stream=None):
        b = budgets.c()
        take = None if take is None else np.ascontiguousarray(take, np.uint32)
        kind = None if kind is None else np.ascontiguousarray(kind, np.uint32)
        level = None if level is None else np.ascontiguousarray(level, np.uint32)
        rb = self._report_buf()
        L.check(L.lib().lc_decode_step(self.h, _ptr(q), _ptr(keys_bf16), _ptr(values_bf16),
                                       C.byref(b), _ptr(take), _ptr(kind), _ptr(level), _ptr(out),
                                       rb.data_ptr(), _stream_ptr(stream)))
        return out

    def decode_step_async(self, q, keys_bf16, values_bf16, budgets: Budgets, take=None, kind=None,
                          level=None, out=None, stream=None):
        """lc_decode_step_async: the same step with take / kind / level as DEVICE
        uint32 tensors [n_slots] (take 0 = no graft on that slot; take None = no
        graft this step).  No host synchronisation: graph-capturable."""
        b = self._budgets_c(budgets)
        rb = self._report_buf()
        L.check(L.lib().lc_decode_step_async(self.h, _ptr(q), _ptr(keys_bf16), _ptr(values_bf16),
                                             C.byref(b), _ptr(take), _ptr(kind), _ptr(level), _ptr(out),
                                             rb.data_ptr(), _stream_ptr(stream)))
        return out

    def compact(self, min_grafted: int = 1, stream=None):
        """lc_compact: grafted chunks into the member CSR (done every 128 decode steps anyway)."""
        L.check(L.lib().lc_compact(self.h, int(min_grafted), _stream_ptr(stream)))

    def _budgets_c(self, budgets: Budgets):
        # keep the ctypes struct alive for the call (and across graph capture)
        self._bc = budgets.c()
        return self._bc

    # ---- evaluator (evaluator.cpp) on the device ----
    def audit_ub(self, slot: int, queries: np.ndarray, tolerance: float = 1e-6) -> int:
        """eval::audit_ub_soundness (evaluator.cpp:107-140) of the slot's live index."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        total = 0
        for i in range(0, q.shape[0], 64):
            part = np.ascontiguousarray(q[i:i + 64])
            v = L.u64()
            L.check(L.lib().lc_audit_ub(self.h, slot, part.ctypes.data, part.shape[0], tolerance, C.byref(v)))
            total += v.value
        return total

    def oracle_topk(self, slot: int, queries: np.ndarray, budget: int) -> np.ndarray:
        """eval::oracle_topk_tokens (evaluator.cpp:43-64) -> [nq, min(budget, n)] sorted ids."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        n = self.slot_dims(slot)[4]
        out = np.zeros((q.shape[0], max(min(budget, n), 1)), np.uint32)
        k = L.u64()
        L.check(L.lib().lc_oracle_topk(self.h, slot, q.ctypes.data, q.shape[0], budget, out.ctypes.data,
                                       C.byref(k)))
        return out[:, : k.value]

    def full_attention(self, slot: int, q, out=None, stream=None):
        """eval::full_attention (evaluator.cpp:11-41) for the slot's query heads; q cuda [G, d]."""
        if out is None:
            out = torch.zeros_like(q)
        L.check(L.lib().lc_full_attention(self.h, slot, _ptr(q), _ptr(out), _stream_ptr(stream)))
        return out

    def step_bytes(self):
        out = np.zeros(4, np.uint64)
        L.check(L.lib().lc_step_bytes(self.h, out.ctypes.data))
        return [int(x) for x in out]

    def launch_count(self) -> int:
        """Kernels the last retrieve launched (selection + attention)."""
        out = np.zeros(1, np.uint32)
        L.check(L.lib().lc_launch_count(self.h, out.ctypes.data))
        return int(out[0])

    def attend_timing(self, arm: int = 0):
        """(summed ms, launches) of the k_attend launches timed since the last
        call (CUDA events around k_attend alone), then arm `arm` more."""
        ms = np.zeros(1, np.float32)
        n = np.zeros(1, np.uint32)
        L.check(L.lib().lc_attend_timing(self.h, arm, ms.ctypes.data, n.ctypes.data))
        return float(ms[0]), int(n[0])

    def device_error(self, clear: bool = True) -> int:
        out = np.zeros(1, np.uint32)
        L.check(L.lib().lc_device_error(self.h, out.ctypes.data, int(clear)))
        return int(out[0])


# ---- host chunker (chunker.cpp:103-149) over the C ABI ----------------------
def _texts(texts: Sequence[str]):
    enc = [t.encode() for t in texts]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    return arr, enc


def segment(texts: Sequence[str], min_len: int = 8, max_len: int = 16) -> np.ndarray:
    arr, keep = _texts(texts)
    out = np.zeros((len(texts) + 1, 4), np.uint32)
    n = L.u64()
    L.check(L.lib().lc_segment(arr, len(texts), min_len, max_len, out.ctypes.data, out.shape[0],
                               C.byref(n)))
    return out[: n.value].copy()


def segment_codes(codes: np.ndarray, min_len: int = 8, max_len: int = 16) -> np.ndarray:
    """segment() over text codes (0 "", 1 "\\n", 2 "}") via packed strings."""
    codes = np.asarray(codes, np.uint8)
    table = {0: b"", 1: b"\n", 2: b"}"}
    lens = np.where(codes == 0, 0, 1).astype(np.uint64)
    offs = np.zeros(len(codes) + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    buf = np.frombuffer(b"".join(table[int(c)] for c in codes[codes != 0]) + b"\0", np.uint8).copy()
    out = np.zeros((len(codes) + 1, 4), np.uint32)
    n = L.u64()
    L.check(L.lib().lc_segment_packed(buf.ctypes.data, offs.ctypes.data, len(codes), min_len, max_len,
                                      out.ctypes.data, out.shape[0], C.byref(n)))
    return out[: n.value].copy()


def flush_take(buffer_texts: Sequence[str], structure_aware=True, min_len=8, max_len=16):
    arr, keep = _texts(buffer_texts)
    t, k, lv = L.u32(), L.u32(), L.u32()
    L.check(L.lib().lc_flush_take(arr, len(buffer_texts), int(structure_aware), min_len, max_len,
                                  C.byref(t), C.byref(k), C.byref(lv)))
    return t.value, k.value, lv.value


# ---- single-head reference-shaped API ---------------------------------------
def _jaccard(a, b):
    # eval::jaccard (evaluator.cpp:75-82); inputs sorted
    if len(a) == 0 and len(b) == 0:
        return 1.0
    sa, sb = set(a.tolist()), set(b.tolist())
    return len(sa & sb) / len(sa | sb)


def _window_hit(history, cur):
    # eval::window_hit (evaluator.cpp:84-95)
    if len(cur) == 0:
        return 1.0
    seen = set()
    for s in history:
        seen.update(s.tolist())
    return sum(1 for x in cur.tolist() if x in seen) / len(cur)


class DeviceIndex:
    """A HierarchicalIndex + TokenStore resident on the GPU (a 1-slot Engine)."""

    def __init__(self, ix: HostIndex, keys: np.ndarray, values: np.ndarray, group: int = 1,
                 extra_tokens: int = 0, extra_chunks: int = 0, structure_aware: bool = True,
                 graft_full: bool = False, device: int = 0, kv_f32: bool = False, pooling: int = 0):
        n = keys.shape[0]
        self.engine = Engine(1, ix.dim, group, cap_tokens=n + extra_tokens + 1,
                             cap_chunks=ix.n_chunks + extra_chunks + 1,
                             cap_clusters=ix.n_clusters, cap_units=max(ix.n_units, 1),
                             structure_aware=structure_aware, graft_full=graft_full, device=device,
                             kv_f32=kv_f32, pooling=pooling)
        self.engine.upload_slot(0, ix, keys, values)
        self.dim = ix.dim
        self.group = group
        self.device = device

    def _q(self, qs):
        q = np.zeros((1, self.group, self.dim), np.float32)
        qs = np.asarray(qs, np.float32).reshape(-1, self.dim)
        q[0, : qs.shape[0]] = qs
        return torch.from_numpy(q).to(f"cuda:{self.device}")

    def retrieve_group(self, qs, budgets: Budgets, buffer_ids=None, with_output=True):
        """retrieve() for up to `group` queries against this index."""
        budgets.validate()
        q = self._q(qs)
        out = torch.zeros_like(q) if with_output else None
        if buffer_ids is not None and len(buffer_ids):
            ids = np.unique(np.asarray(buffer_ids, np.uint32))
            n = self.engine.slot_dims(0)[4]
            if ids.size and ids.max() >= n:
                raise ValueError("buffer id beyond the token store")
            bo = torch.tensor([0, len(ids)], dtype=torch.int32, device=q.device)
            bi = torch.from_numpy(ids.astype(np.int32)).to(q.device)
            self.engine.retrieve(q, budgets, "list", out=out, buf_off=bo, buf_ids=bi)
        else:
            self.engine.retrieve(q, budgets, "none", out=out)
        o = out.cpu().numpy()[0] if with_output else None
        res = []
        for g in range(np.asarray(qs).reshape(-1, self.dim).shape[0]):
            r = self.engine.selection(0, g, active=True)
            r.output = None if o is None else o[g].copy()
            res.append(r)
        return res


def retrieve(index: DeviceIndex, q, budgets: Budgets, buffer_ids=()) -> RetrievalResult:
    """retrieve() (retriever.hpp:49-51)."""
    return index.retrieve_group(q, budgets, buffer_ids, True)[0]


def retrieve_ids(index: DeviceIndex, q, budgets: Budgets, buffer_ids=()) -> RetrievalResult:
    """retrieve_ids() (retriever.hpp:53-55): selection only, output left empty."""
    return index.retrieve_group(q, budgets, buffer_ids, False)[0]


class StreamState:
    """StreamState (streamer.hpp:47-85) over a 1-slot engine.

    Tokens are (id, text, key, value); the step's attention runs before the
    token enters the store (streamer.cpp:149-163), and a chunk is carved and
    grafted when the buffer reaches max_len."""

    def __init__(self, ix: HostIndex, keys: np.ndarray, values: np.ndarray, texts: Sequence[str],
                 structure_aware=True, graft_full=False, extra_tokens=4096, extra_chunks=512,
                 history_capacity=32, min_len=8, max_len=16, device=0, group=1, pooling=0):
        self.index = DeviceIndex(ix, keys, values, group=group, extra_tokens=extra_tokens,
                                 extra_chunks=extra_chunks, structure_aware=structure_aware,
                                 graft_full=graft_full, device=device, pooling=pooling)
        self.engine = self.index.engine
        self.texts = list(texts)
        self.structure_aware = structure_aware
        self.min_len, self.max_len = min_len, max_len
        self.history: deque = deque()
        self.history_capacity = history_capacity
        self.graft_count = 0
        self.device = device

    @property
    def n_tokens(self):
        return self.engine.slot_dims(0)[4]

    @property
    def chunked_end(self):
        return self.engine.slot_dims(0)[7]

    def buffer_size(self):
        return self.n_tokens - self.chunked_end

    def buffer_ids(self):
        return np.arange(self.chunked_end, self.n_tokens, dtype=np.uint32)

    def _append(self, token_id, text, key, value):
        if token_id != self.n_tokens:  # TokenStore::append (types.hpp:38-39)
            raise ValueError("non-sequential token id")
        k = torch.from_numpy(bf16_bits(np.asarray(key, np.float32)[None]).view(np.int16)).to(f"cuda:{self.device}")
        v = torch.from_numpy(bf16_bits(np.asarray(value, np.float32)[None]).view(np.int16)).to(f"cuda:{self.device}")
        self.texts.append(text)
        return k, v

    def _flush(self):
        buf = self.texts[self.chunked_end:]
        return flush_take(buf, self.structure_aware, self.min_len, self.max_len)

    def push_token(self, token_id, text, key, value) -> Optional[GraftReport]:
        """push_token + graft_chunk of the emitted chunk (streamer.cpp:56-66, 68-143)."""
        k, v = self._append(token_id, text, key, value)
        self.engine.kv_append(k, v)
        if self.buffer_size() >= self.max_len:
            take, kind, level = self._flush()
            self.engine.graft(np.array([take], np.uint32), np.array([kind], np.uint32),
                              np.array([level], np.uint32))
            self.graft_count += 1
            return self._report()
        return None

    def _report(self):
        r = self.engine.reports()[0]
        return GraftReport(int(r["chunk_id"]), int(r["cluster_id"]), int(r["unit_id"]),
                           float(r["centroid_delta"]), float(r["fine_radius"]),
                           float(r["coarse_radius"]), int(r["distance_comps"]))

    def decode_step(self, q, token_id, text, key, value, budgets: Budgets) -> DecodeOutcome:
        """decode_step (streamer.cpp:145-165)."""
        budgets.validate()
        qd = self.index._q(q)
        out = torch.zeros_like(qd)
        k, v = self._append(token_id, text, key, value)
        # the flush decision is known before the step: buffer after the push
        take = np.zeros(1, np.uint32)
        kind = np.zeros(1, np.uint32)
        level = np.zeros(1, np.uint32)
        if self.buffer_size() + 1 >= self.max_len:
            buf = self.texts[self.chunked_end:]
            t, kd, lv = flush_take(buf, self.structure_aware, self.min_len, self.max_len)
            take[0], kind[0], level[0] = t, kd, lv
        self.engine.decode_step(qd, k, v, budgets, take, kind, level, out)
        r = self.engine.selection(0, 0, active=True)
        r.output = out.cpu().numpy()[0, 0].copy()
        sel = np.sort(r.selected_clusters)
        outcome = DecodeOutcome(r)
        outcome.jaccard = _jaccard(self.history[-1] if self.history else np.zeros(0, np.uint32), sel)
        outcome.window_hit = _window_hit(list(self.history), sel)
        self.history.append(sel)
        while len(self.history) > self.history_capacity:
            self.history.popleft()
        if take[0]:
            self.graft_count += 1
            outcome.graft = self._report()
        return outcome
