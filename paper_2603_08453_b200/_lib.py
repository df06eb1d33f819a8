"""ctypes binding of the C ABI (include/lychee_b200.h) -> liblychee_b200.so.

The product path is this library; there is no CPU or eager fallback.  Loading
fails loudly when the in-tree .so is missing.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LC_LIB_PATH") or os.path.join(PKG, "liblychee_b200.so")  # override: A/B runs only

LC_OK, LC_EINVAL, LC_ERUNTIME, LC_ECUDA, LC_ENOMEM = 0, 1, 2, 3, 4
LC_BUFFER_NONE, LC_BUFFER_STREAM, LC_BUFFER_LIST = 0, 1, 2

vp = C.c_void_p
u32 = C.c_uint32
u64 = C.c_uint64


class IndexDesc(C.Structure):
    _fields_ = [("n_slots", u32), ("dim", u32), ("group", u32), ("cap_tokens", u32),
                ("cap_chunks", u32), ("cap_clusters", u32), ("cap_units", u32),
                ("max_candidates", u32), ("structure_aware", u32),
                ("graft_full", u32), ("keep_reps", u32), ("pooling", u32), ("slot_groups", u32),
                ("device", C.c_int32), ("kv_f32", u32)]


class Budgets_(C.Structure):
    _fields_ = [("unit_topk", u32), ("mode", u32), ("cluster_topk", u32), ("token_budget", u64),
                ("sink_size", u32)]


class HostIndex_(C.Structure):
    _fields_ = [("dim", u32), ("n_chunks", u32), ("n_clusters", u32), ("n_units", u32),
                ("chunk_span", vp), ("chunk_rep", vp), ("fine_centroid", vp), ("fine_radius", vp),
                ("fine_token_count", vp), ("fine_parent", vp), ("fine_member_off", vp),
                ("fine_members", vp), ("coarse_centroid", vp), ("coarse_radius", vp),
                ("coarse_member_off", vp), ("coarse_members", vp), ("cluster_of_chunk", vp)]


class IndexConfig_(C.Structure):
    _fields_ = [("avg_chunks_per_cluster", C.c_double), ("max_coarse_units", u32),
                ("kmeans_iters", u32), ("pooling", u32), ("elem_bytes", u32), ("seed", u64)]


class GraftReport_(C.Structure):
    _fields_ = [("chunk_id", u32), ("cluster_id", u32), ("unit_id", u32), ("_pad", u32),
                ("centroid_delta", C.c_double), ("fine_radius", C.c_double),
                ("coarse_radius", C.c_double), ("distance_comps", u64)]


class SelectionInfo_(C.Structure):
    _fields_ = [("n_units", u32), ("n_clusters", u32), ("degenerate", u32), ("error", u32),
                ("scanned_centroids", u64), ("n_active", u64)]


# every symbol include/lychee_b200.h declares
EXPORTS = [
    "lc_last_error", "lc_index_create", "lc_index_destroy", "lc_index_get_desc",
    "lc_index_upload_slot", "lc_index_slot_dims", "lc_index_download_slot", "lc_cluster_download", "lc_kv_append",
    "lc_kv_upload_slot", "lc_kv_download_slot",
    "lc_retrieve", "lc_retrieve_slots", "lc_set_gather", "lc_gather_wait", "lc_sparse_attention", "lc_graft", "lc_decode_step", "lc_decode_step_async", "lc_compact", "lc_retrieve_host",
    "lc_selection_download", "lc_selection_stage", "lc_selection_read_staged", "lc_step_bytes", "lc_launch_count", "lc_attend_timing", "lc_device_error", "lc_segment", "lc_segment_packed", "lc_flush_take",
    "lc_index_build", "lc_gen_workload", "lc_graft_rep", "lc_sparse_attention_ids", "lc_chunk_rep",
    "lc_index_set_config", "lc_index_get_config", "lc_index_to_bytes", "lc_index_save", "lc_index_load",
    "lc_tkix_encode", "lc_tkix_decode_dims", "lc_tkix_decode",
    "lc_audit_ub", "lc_oracle_topk", "lc_full_attention",
]

_lib = None


class LcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class LcInvalidArgument(LcError, ValueError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"native library missing: {LIB_PATH}; run python -m paper_2603_08453_b200._build "
                "(there is no fallback path)")
        L = C.CDLL(LIB_PATH)
        L.lc_last_error.restype = C.c_char_p
        L.lc_index_create.argtypes = [C.POINTER(IndexDesc), C.POINTER(vp)]
        L.lc_index_destroy.argtypes = [vp]
        L.lc_index_destroy.restype = None
        L.lc_index_get_desc.argtypes = [vp, C.POINTER(IndexDesc)]
        L.lc_index_upload_slot.argtypes = [vp, u32, C.POINTER(HostIndex_), vp, vp, u32]
        L.lc_index_slot_dims.argtypes = [vp, u32, vp]
        L.lc_index_download_slot.argtypes = [vp, u32, C.POINTER(HostIndex_)]
        L.lc_kv_append.argtypes = [vp, vp, vp, vp]
        L.lc_kv_upload_slot.argtypes = [vp, u32, vp, vp, u32]
        L.lc_kv_download_slot.argtypes = [vp, u32, vp, vp, u32]
        L.lc_retrieve.argtypes = [vp, vp, C.POINTER(Budgets_), u32, vp, vp, vp, vp]
        L.lc_retrieve_slots.argtypes = [vp, u32, u32, vp, C.POINTER(Budgets_), u32, vp, vp, vp, vp]
        L.lc_set_gather.argtypes = [vp, u32, vp, vp, vp, C.c_uint64, u32]
        L.lc_gather_wait.argtypes = [vp, vp]
        L.lc_sparse_attention.argtypes = [vp, vp, vp, vp]
        L.lc_graft.argtypes = [vp, vp, vp, vp, vp, vp]
        L.lc_decode_step.argtypes = [vp, vp, vp, vp, C.POINTER(Budgets_), vp, vp, vp, vp, vp, vp]
        L.lc_compact.argtypes = [vp, u32, vp]
        L.lc_decode_step_async.argtypes = [vp, vp, vp, vp, C.POINTER(Budgets_), vp, vp, vp, vp, vp, vp]
        L.lc_retrieve_host.argtypes = [vp, vp, C.POINTER(Budgets_), u32, vp, vp]
        L.lc_selection_stage.argtypes = [vp, u32, u32, vp]
        L.lc_selection_read_staged.argtypes = [vp, C.POINTER(SelectionInfo_), vp, u64, vp, u64, vp, u64]
        L.lc_selection_download.argtypes = [vp, u32, u32, C.POINTER(SelectionInfo_), vp, u64, vp,
                                            u64, vp, u64]
        L.lc_step_bytes.argtypes = [vp, vp]
        L.lc_launch_count.argtypes = [vp, vp]
        L.lc_attend_timing.argtypes = [vp, u32, vp, vp]
        L.lc_device_error.argtypes = [vp, vp, C.c_int]
        L.lc_segment.argtypes = [vp, u32, u32, u32, vp, u64, C.POINTER(u64)]
        L.lc_segment_packed.argtypes = [vp, vp, u32, u32, u32, vp, u64, C.POINTER(u64)]
        L.lc_flush_take.argtypes = [vp, u32, u32, u32, u32, C.POINTER(u32), C.POINTER(u32),
                                    C.POINTER(u32)]
        L.lc_index_build.argtypes = [vp, vp, vp, vp, C.c_double, u32, u32, vp]
        L.lc_gen_workload.argtypes = [vp, u32, u32, C.c_double, u32, C.c_double, vp, vp, vp]
        L.lc_graft_rep.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.lc_sparse_attention_ids.argtypes = [vp, u32, vp, vp, u32, vp, vp]
        L.lc_chunk_rep.argtypes = [vp, u32, u32, u32, vp]
        L.lc_index_set_config.argtypes = [vp, u32, C.POINTER(IndexConfig_)]
        L.lc_index_get_config.argtypes = [vp, u32, C.POINTER(IndexConfig_)]
        L.lc_index_to_bytes.argtypes = [vp, u32, vp, u64, C.POINTER(u64)]
        L.lc_index_save.argtypes = [vp, u32, C.c_char_p, vp, vp]
        L.lc_index_load.argtypes = [vp, u32, C.c_char_p, vp, u64, vp, u64, C.POINTER(u64)]
        L.lc_tkix_encode.argtypes = [C.POINTER(HostIndex_), C.POINTER(IndexConfig_), vp, u64, C.POINTER(u64)]
        L.lc_tkix_decode_dims.argtypes = [vp, u64, vp]
        L.lc_tkix_decode.argtypes = [vp, u64, C.POINTER(HostIndex_), C.POINTER(IndexConfig_)]
        L.lc_audit_ub.argtypes = [vp, u32, vp, u32, C.c_double, C.POINTER(u64)]
        L.lc_oracle_topk.argtypes = [vp, u32, vp, u32, u64, vp, C.POINTER(u64)]
        L.lc_full_attention.argtypes = [vp, u32, vp, vp, vp]
        _lib = L
    return _lib


def check(rc: int):
    if rc == LC_OK:
        return
    msg = lib().lc_last_error().decode(errors="replace")
    if rc == LC_EINVAL:
        raise LcInvalidArgument(rc, msg)
    raise LcError(rc, msg)
