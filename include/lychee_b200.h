/* lychee_b200.h -- C ABI of the B200-native LycheeCluster decode-step path.
 *
 * Drop-in boundary for the reference's per-decode-step retrieval + sparse
 * attention + lazy graft (reference: /root/reference/proj, library `tierkv`).
 * Plain C: opaque handles, plain pointers and sizes, int status codes, no
 * exceptions and no C++/torch types cross it.  Device pointers are CUDA
 * device addresses; `stream` is a cudaStream_t passed as void*.
 *
 * One handle owns every "slot" resident on one GPU.  A slot is one
 * (layer, KV head, sequence) triple: its own TokenStore K/V, its own
 * HierarchicalIndex and its own stream cursor -- the reference's single-head
 * engine instanced per KV head.  A GQA group of `group` query
 * heads is scored against its KV head's slot; query head g of slot s is the
 * reference call retrieve(index[s], q[s][g], budgets, buffer) (retriever.hpp:49).
 *
 * Status codes: 0 ok; LC_EINVAL = std::invalid_argument in the reference;
 * LC_ERUNTIME = std::runtime_error; LC_ECUDA; LC_ENOMEM.  lc_last_error()
 * returns the thread-local message of the last failure.
 */
#ifndef LYCHEE_B200_H
#define LYCHEE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LC_OK 0
#define LC_EINVAL 1
#define LC_ERUNTIME 2
#define LC_ECUDA 3
#define LC_ENOMEM 4

#define LC_MODE_FIXED_CLUSTER_COUNT 0 /* SelectionMode::fixed_cluster_count */
#define LC_MODE_TOKEN_BUDGET 1        /* SelectionMode::token_budget */

/* retrieve flags */
#define LC_BUFFER_NONE 0u   /* buffer_ids = {} (retriever.hpp:52 default) */
#define LC_BUFFER_STREAM 1u /* buffer_ids = StreamState::buffer_ids() = [chunked_end, n) (streamer.cpp:23-27) */
#define LC_BUFFER_LIST 2u   /* explicit per-slot id lists (see lc_retrieve) */

typedef struct lc_index_s* lc_index_t;

/* Engine shape.  Replaces the reference's per-head objects
 * (TokenStore types.hpp:25-57, HierarchicalIndex index.hpp:60-73,
 * StreamerConfig streamer.hpp:19-25) with one HBM-resident SoA arena. */
typedef struct {
    uint32_t n_slots;         /* layers x KV heads x sequences */
    uint32_t dim;             /* head dim d (attention kernel: 64 or 128) */
    uint32_t group;           /* GQA query heads per slot: 1, 2, 4 or 8 */
    uint32_t cap_tokens;      /* per-slot KV capacity (prefix + decode) */
    uint32_t cap_chunks;      /* per-slot chunk capacity (prefill + grafts) */
    uint32_t cap_clusters;    /* per-slot fine clusters L (fixed after build) */
    uint32_t cap_units;       /* per-slot coarse units P (<= 1024) */
    uint32_t max_candidates;  /* bound on fine candidates per query (0 = auto) */
    uint32_t structure_aware; /* StreamerConfig::structure_aware (host chunker) */
    uint32_t graft_full;      /* StreamerConfig::graft_search == full */
    uint32_t keep_reps;       /* keep chunk representatives on device (download parity) */
    uint32_t pooling;         /* IndexConfig::pooling: 0 mean, 1 max (index.hpp:11) */
    uint32_t slot_groups;     /* lc_retrieve runs this many slot groups on forked streams so
                                 one group's selection overlaps another's attention (0 = 1) */
    int32_t device;
    uint32_t kv_f32;          /* 0: K/V in bf16 (the bench / serving layout; dim 64 or 128);
                                 1: fp32 K/V exactly as the reference's TokenStore, attention
                                 in fp64 (reference-exact mode; dim 8/16/32 also allowed for
                                 group 1 or 4) */
} lc_index_desc;

/* tierkv::Budgets (retriever.hpp:13-21) */
typedef struct {
    uint32_t unit_topk;
    uint32_t mode;
    uint32_t cluster_topk;
    uint64_t token_budget;
    uint32_t sink_size;
} lc_budgets;

/* Host view of one tierkv::HierarchicalIndex in the reference's own numbering
 * (index.hpp:25-73); member lists as CSR.  Used for upload and download. */
typedef struct {
    uint32_t dim, n_chunks, n_clusters, n_units;
    uint32_t* chunk_span;        /* [n_chunks*4] start, end, kind, level */
    float* chunk_rep;            /* [n_chunks*dim] (may be NULL on upload) */
    float* fine_centroid;        /* [n_clusters*dim] */
    double* fine_radius;         /* [n_clusters] */
    uint64_t* fine_token_count;  /* [n_clusters] */
    uint32_t* fine_parent;       /* [n_clusters] */
    uint32_t* fine_member_off;   /* [n_clusters+1] */
    uint32_t* fine_members;      /* chunk ids */
    float* coarse_centroid;      /* [n_units*dim] */
    double* coarse_radius;       /* [n_units] */
    uint32_t* coarse_member_off; /* [n_units+1] */
    uint32_t* coarse_members;    /* fine ids, ascending within a unit */
    uint32_t* cluster_of_chunk;  /* [n_chunks] */
} lc_host_index;

/* tierkv::IndexConfig (index.hpp:13-22): recorded per slot (defaults at
 * upload, the build's parameters after lc_index_build, the file's after
 * lc_index_load) and serialized by index_to_bytes. */
typedef struct {
    double avg_chunks_per_cluster; /* 2.0 */
    uint32_t max_coarse_units;     /* 64 */
    uint32_t kmeans_iters;         /* 10 */
    uint32_t pooling;              /* 0 mean, 1 max */
    uint32_t elem_bytes;           /* 2 */
    uint64_t seed;                 /* 0 */
} lc_index_config;

/* tierkv::GraftReport (streamer.hpp:27-35) */
typedef struct {
    uint32_t chunk_id, cluster_id, unit_id, _pad;
    double centroid_delta, fine_radius, coarse_radius;
    uint64_t distance_comps;
} lc_graft_report;

/* Per query head selection summary (RetrievalResult minus the id lists). */
typedef struct {
    uint32_t n_units, n_clusters, degenerate, error;
    uint64_t scanned_centroids; /* RetrievalResult::scanned_centroids */
    uint64_t n_active;          /* |active_token_ids| */
} lc_selection_info;

const char* lc_last_error(void);

/* Allocate every slot's arena on desc->device.  Replaces constructing
 * H x layers tierkv::StreamState objects (streamer.hpp:49). */
int lc_index_create(const lc_index_desc* desc, lc_index_t* out);
void lc_index_destroy(lc_index_t h);
int lc_index_get_desc(lc_index_t h, lc_index_desc* out);

/* Upload one slot: a HierarchicalIndex produced by build_index (index.hpp:93-95)
 * plus its TokenStore keys/values (host memory, bf16 bit patterns or fp32 as
 * desc.kv_f32 says), n_tokens rows.  The stream cursor starts at chunked_end = last chunk end
 * (streamer.cpp:13-21), so tokens past it form the buffer.  Replaces
 * StreamState::StreamState(TokenStore, HierarchicalIndex, StreamerConfig).
 * keys_bf16 == values_bf16 == NULL keeps the K/V already resident in the slot
 * (e.g. written by lc_gen_workload). */
int lc_index_upload_slot(lc_index_t h, uint32_t slot, const lc_host_index* ix,
                         const void* keys, const void* values, uint32_t n_tokens);

/* Sizes of a slot's current index: dims[0..7] = dim, n_chunks, n_clusters,
 * n_units, n_tokens, total fine members, total coarse members, chunked_end. */
int lc_index_slot_dims(lc_index_t h, uint32_t slot, uint64_t* dims);

/* Download a slot's index back into the reference layout, including every
 * graft applied on the device (for index_to_bytes parity, serialize.cpp:88-125).
 * Caller allocates every array from lc_index_slot_dims.  Synchronous. */
int lc_index_download_slot(lc_index_t h, uint32_t slot, lc_host_index* out);

/* One fine cluster of a slot in the reference numbering: FineCluster::centroid
 * [dim], radius, token_count (any pointer may be NULL).  A graft changes one
 * cluster, one unit and appends one chunk (streamer.cpp:108-134), so a host
 * mirror (the C++ drop-in's HierarchicalIndex) is patched from the graft
 * report plus this call instead of re-downloading the index.  Synchronous. */
int lc_cluster_download(lc_index_t h, uint32_t slot, uint32_t cluster_id, float* centroid,
                        double* radius, uint64_t* token_count);

/* Raw K/V rows of one slot (host memory, element type per desc.kv_f32): write rows
 * [0, n_tokens) and set the slot's store size (the index is left as is), or
 * read them back.  TokenStore::keys_flat/values_flat (types.hpp:48-49). */
int lc_kv_upload_slot(lc_index_t h, uint32_t slot, const void* keys, const void* values,
                      uint32_t n_tokens);
int lc_kv_download_slot(lc_index_t h, uint32_t slot, void* keys, void* values, uint32_t n_tokens);

/* Append one decoded token's K/V (device [n_slots][dim] each, element type per
 * desc.kv_f32) to every slot -- TokenStore::append inside push_token
 * (streamer.cpp:56-58). */
int lc_kv_append(lc_index_t h, const void* keys_dev, const void* values_dev, void* stream);

/* Batched retrieve() over every query head of every slot (retriever.cpp:161-167):
 * coarse UB scoring + top-k_g, fine UB scoring, selection (fixed k_c or greedy
 * token-budget prefix fill), active-set construction and -- when out_dev is
 * non-NULL -- sparse attention (retriever.cpp:41-50) into out_dev
 * [n_slots][group][dim] fp32.  q_dev: [n_slots][group][dim] fp32.
 * flags: LC_BUFFER_*; for LC_BUFFER_LIST, buf_off_dev [n_slots+1] and
 * buf_ids_dev (sorted, unique, < n_tokens per slot) give each slot's ids.
 * Asynchronous on `stream`. */
int lc_retrieve(lc_index_t h, const float* q_dev, const lc_budgets* b, uint32_t flags,
                const uint32_t* buf_off_dev, const uint32_t* buf_ids_dev, float* out_dev,
                void* stream);

/* lc_retrieve over the slot range [first_slot, first_slot + n_slots) only
 * (q_dev / out_dev keep the handle-wide [n_slots][group][dim] layout; rows
 * outside the range are neither read nor written): one layer's KV heads of a
 * layer-by-layer decode, whose head outputs are gathered across GPUs at the
 * layer boundary before the next layer's queries exist. */
int lc_retrieve_slots(lc_index_t h, uint32_t first_slot, uint32_t n_slots, const float* q_dev,
                      const lc_budgets* b, uint32_t flags, const uint32_t* buf_off_dev,
                      const uint32_t* buf_ids_dev, float* out_dev, void* stream);

/* Fused all-gather epilogue: the layer-boundary exchange
 * of head outputs done by the attention merge itself.  After this call every
 * merged (slot, head) output row of lc_retrieve / lc_retrieve_slots /
 * lc_decode_step* is also stored into each of the n_peers gather buffers
 * (peer_out[r]: a device pointer valid in this process -- NVLink peer memory
 * of rank r, e.g. a symmetric-memory / IPC mapping -- laid out
 * [rows][group][dim] fp32, this handle's slot s at row row_of_slot[s]), and
 * each peer's uint32 arrival counter peer_flag[r] is incremented once per row
 * (system-scope atomics after a system fence).  lc_gather_wait then blocks
 * the stream until this rank's own counter (my_flag) has advanced by
 * rows_per_wait since the previous wait -- every rank's rows of the step or
 * layer have landed.  The wait count lives on the device, so the pair is
 * CUDA-graph capturable.  n_peers = 0 turns the epilogue off.  peer_out /
 * peer_flag / row_of_slot are host arrays (copied). */
int lc_set_gather(lc_index_t h, uint32_t n_peers, const uint64_t* peer_out, const uint64_t* peer_flag,
                  const uint32_t* row_of_slot, uint64_t my_flag, uint32_t rows_per_wait);
int lc_gather_wait(lc_index_t h, void* stream);

/* Sparse attention over the active sets of the last lc_retrieve (the second
 * half of retrieve(), retriever.cpp:165). */
int lc_sparse_attention(lc_index_t h, const float* q_dev, float* out_dev, void* stream);

/* Lazy incremental update: for every slot with take[slot] > 0, carve the chunk
 * [chunked_end, chunked_end + take) (flush_buffer, streamer.cpp:29-54; the host
 * decides `take` with the chunker, kind/level are recorded for download), pool
 * its representative (index.cpp:20-41) and graft it (graft_chunk,
 * streamer.cpp:68-143).  take/kind/level: host arrays [n_slots].  reports_dev:
 * device [n_slots] (entries of slots without a graft are left untouched). */
int lc_graft(lc_index_t h, const uint32_t* take, const uint32_t* kind, const uint32_t* level,
             lc_graft_report* reports_dev, void* stream);

/* One StreamState::decode_step for every slot (streamer.cpp:145-165):
 * retrieve + attend with buffer_ids = [chunked_end, n), then append the step's
 * token, then graft where take[slot] > 0.  Stability metrics (jaccard /
 * window_hit) are host bookkeeping and stay in the caller. */
int lc_decode_step(lc_index_t h, const float* q_dev, const void* keys_dev,
                   const void* values_dev, const lc_budgets* b, const uint32_t* take,
                   const uint32_t* kind, const uint32_t* level, float* out_dev,
                   lc_graft_report* reports_dev, void* stream);

/* lc_decode_step with take / kind / level as DEVICE arrays [n_slots] (take 0:
 * no graft on that slot; take_dev NULL: no graft this step) and no host
 * synchronisation or host bookkeeping: every launch reads the stream cursors
 * from the device, so a run of steps can be captured in one CUDA graph
 * (config 3).  Device-side checks replace the host ones (sticky error bits:
 * token / chunk capacity, take outside the buffered tokens).  The handle's
 * host view of the cursors is refreshed from the device, synchronously, by
 * the next call that needs it (download, graft, TKIX, ...). */
int lc_decode_step_async(lc_index_t h, const float* q_dev, const void* keys_dev,
                         const void* values_dev, const lc_budgets* b, const uint32_t* take_dev,
                         const uint32_t* kind_dev, const uint32_t* level_dev, float* out_dev,
                         lc_graft_report* reports_dev, void* stream);

/* Chunk-table compaction: fold every slot's grafted chunks (those appended
 * since the last compaction) into the cluster member lists the selection
 * reads, for slots with at least min_grafted of them.  lc_decode_step and
 * lc_decode_step_async do it on their own every 128 steps; member order and
 * every downloaded / serialized field are unchanged.  LC_EINVAL when the
 * chunk table exceeds the kernel's shared-memory staging (~1M-token slots). */
int lc_compact(lc_index_t h, uint32_t min_grafted, void* stream);

/* graft_chunk(Chunk) (streamer.cpp:68-143) with the chunk's representative
 * supplied by the caller instead of pooled from the keys: reps_host
 * [n_slots][dim] fp32 (rows of slots without a graft are ignored). */
int lc_graft_rep(lc_index_t h, const uint32_t* take, const uint32_t* kind, const uint32_t* level,
                 const float* reps_host, lc_graft_report* reports_dev, void* stream);

/* chunk_representative (index.cpp:20-41) of rows [start, start + take) of a
 * slot's store, pooled with desc.pooling, into rep_host [dim].  A zero norm is
 * LC_ERUNTIME, as the reference throws std::runtime_error.  Synchronous. */
int lc_chunk_rep(lc_index_t h, uint32_t slot, uint32_t start, uint32_t take, float* rep_host);

/* sparse_attention(q, store, ids) (retriever.cpp:41-50) for one slot over an
 * explicit id list (host, each < the slot's token count): q_dev [group][dim]
 * for the slot's query heads, out_dev [group][dim].  Empty lists are
 * LC_EINVAL, as the reference throws.  Overwrites the slot's active row list,
 * so lc_sparse_attention needs a fresh lc_retrieve afterwards.  Synchronous. */
int lc_sparse_attention_ids(lc_index_t h, uint32_t slot, const float* q_dev, const uint32_t* ids_host,
                            uint32_t n_ids, float* out_dev, void* stream);

/* End-to-end variant of lc_retrieve over HOST buffers (pinned or pageable):
 * H2D of q, retrieve + attention, D2H of out; synchronous on `stream`. */
int lc_retrieve_host(lc_index_t h, const float* q_host, const lc_budgets* b, uint32_t flags,
                     float* out_host, void* stream);

/* Read back the last selection of query head (slot, g): summary, selected
 * units (rank order), selected clusters (reference ids, rank order) and,
 * optionally, the sorted unique active token ids.  Synchronous. */
int lc_selection_download(lc_index_t h, uint32_t slot, uint32_t g, lc_selection_info* info,
                          uint32_t* units, uint64_t units_cap, uint32_t* clusters,
                          uint64_t clusters_cap, uint32_t* active, uint64_t active_cap);

/* The same result without device-wide synchronisation: lc_selection_stage
 * queues D2H copies of head g of `slot`'s selection (error bits, summary,
 * units, clusters, the slot's spans) into handle-owned page-locked memory on
 * `stream`; after the caller has synchronised that stream,
 * lc_selection_read_staged unpacks them exactly as lc_selection_download
 * would (the C++ drop-in's per-call path: one stream sync per retrieve). */
int lc_selection_stage(lc_index_t h, uint32_t slot, uint32_t g, void* stream);
int lc_selection_read_staged(lc_index_t h, lc_selection_info* info, uint32_t* units, uint64_t units_cap,
                             uint32_t* clusters, uint64_t clusters_cap, uint32_t* active, uint64_t active_cap);

/* Bytes read by the last lc_retrieve in algorithmic terms,
 * computed on the device from the step's own selections: out[0] = union
 * bytes, out[1] = per-query (non-deduplicated) bytes, out[2] = active tokens
 * (union over each slot's group), out[3] = fine candidates (union). Synchronous. */
int lc_step_bytes(lc_index_t h, uint64_t* out);

/* Kernel launches the last lc_retrieve / lc_retrieve_host / lc_decode_step
 * made for selection + attention (k_select or the four-kernel chain, then
 * k_attend + k_merge); the bench's gpu_launches claim. */
int lc_launch_count(lc_index_t h, uint32_t* out);

/* Measurement hook for the bench's per-kernel roofline: reports the summed
 * CUDA-event time (ms) and count of the k_attend launches timed since the
 * previous call (ms_sum / timed may be null), then arms n_launches event
 * pairs: each following single-launch lc_sparse_attention records one pair
 * on its stream around k_attend alone (k_merge follows the second record).
 * n_launches = 0 disarms.  Synchronous when reporting. */
int lc_attend_timing(lc_index_t h, uint32_t n_launches, float* ms_sum, uint32_t* timed);

/* Sticky device-side error bits (lc_common.cuh ErrBits) of every kernel since
 * the last clear; synchronous.  Bit 0 candidates over capacity, 1 empty
 * candidate set (select_topk k = 0), 2 spans over capacity, 3 zero-norm
 * chunk representative, 4 chunk capacity, 5 token capacity, 6 empty active
 * set, 7 graft take outside the buffered tokens, 8 fused all-gather: a peer's
 * rows never arrived, 9 streamed-attention task queue overflow, 10
 * streamed attention: a slot's tasks never published (bounded wait). */
int lc_device_error(lc_index_t h, uint32_t* out, int clear);

/* ---- TKIX <-> device (serialize.cpp:88-220) ------ */

/* IndexConfig of a slot (serialized by index_to_bytes). */
int lc_index_set_config(lc_index_t h, uint32_t slot, const lc_index_config* cfg);
int lc_index_get_config(lc_index_t h, uint32_t slot, lc_index_config* cfg);

/* index_to_bytes(state.index()) (serialize.cpp:88-125) of a slot's live index,
 * every graft included (needs the chunk representatives: keep_reps or an
 * upload that supplied them).  *size = full size; up to cap bytes copied to
 * buf (NULL: size only).  Synchronous. */
int lc_index_to_bytes(lc_index_t h, uint32_t slot, uint8_t* buf, uint64_t cap, uint64_t* size);

/* save_index (serialize.cpp:127-148): a TKIX file of the slot's index plus
 * its token store (texts packed as text_buf[text_offs[i], text_offs[i+1]),
 * NULL = empty texts; K/V as fp32, bf16 stores widened exactly).  The
 * reference's load_index reads it. */
int lc_index_save(lc_index_t h, uint32_t slot, const char* path, const char* text_buf, const uint64_t* text_offs);

/* load_index (serialize.cpp:150-220) into a slot: index + token store
 * uploaded (bf16 engines round K/V to nearest even), IndexConfig recorded.
 * Texts are returned packed when text_buf / text_offs are given (offs needs
 * n_tokens + 1 entries; nothing past the caps is written); *n_tokens = the
 * store size.  Reads files written by the reference's save_index. */
int lc_index_load(lc_index_t h, uint32_t slot, const char* path, char* text_buf, uint64_t text_cap,
                  uint64_t* text_offs, uint64_t offs_cap, uint64_t* n_tokens);

/* Host-only codec of the index part (no device needed): index_to_bytes of a
 * host index, its inverse, and the sizes to allocate for the inverse
 * (dims as lc_index_slot_dims; dims[7] = bytes consumed). */
int lc_tkix_encode(const lc_host_index* ix, const lc_index_config* cfg, uint8_t* buf, uint64_t cap,
                   uint64_t* size);
int lc_tkix_decode_dims(const uint8_t* buf, uint64_t size, uint64_t* dims);
int lc_tkix_decode(const uint8_t* buf, uint64_t size, lc_host_index* out, lc_index_config* cfg);

/* ---- evaluator on the device (evaluator.cpp) ------ */

/* eval::audit_ub_soundness (evaluator.cpp:107-140) of one slot's live index
 * for nq <= 64 host queries [nq][dim]: the number of (query, tier node,
 * descendant chunk) triples whose exact rep dot exceeds the node's bound +
 * tolerance -- the reference's count, bit for bit.  Needs keep_reps. */
int lc_audit_ub(lc_index_t h, uint32_t slot, const float* queries_host, uint32_t nq, double tolerance,
                uint64_t* violations);

/* eval::oracle_topk_tokens (evaluator.cpp:43-64) over the slot's whole store
 * for nq host queries: ids_out [nq][min(budget, n)] sorted ascending, ties
 * toward the smaller id; *n_out = min(budget, n).  budget 0 is LC_EINVAL. */
int lc_oracle_topk(lc_index_t h, uint32_t slot, const float* queries_host, uint32_t nq, uint64_t budget,
                   uint32_t* ids_out, uint64_t* n_out);

/* eval::full_attention (evaluator.cpp:11-41) over the slot's whole store for
 * its `group` query heads: q_dev [group][dim] -> out_dev [group][dim]
 * (bf16 store: fp32 accumulation; kv_f32: fp64).  Asynchronous; overwrites
 * the slot's active row list like lc_sparse_attention_ids. */
int lc_full_attention(lc_index_t h, uint32_t slot, const float* q_dev, float* out_dev, void* stream);

/* ---- host chunk-boundary decision (streaming front end) ----------------- */

/* segment() with ChunkPolicy::defaults()'s separator table and the given
 * min/max lengths (chunker.cpp:103-149).  spans4: start, end, kind
 * (0 natural, 1 forced, 2 tail), level; up to cap spans. */
int lc_segment(const char* const* texts, uint32_t n, uint32_t min_len, uint32_t max_len,
               uint32_t* spans4, uint64_t cap, uint64_t* n_spans);

/* lc_segment over packed texts: text i = buf[offs[i], offs[i+1]). */
int lc_segment_packed(const char* buf, const uint64_t* offs, uint32_t n, uint32_t min_len,
                      uint32_t max_len, uint32_t* spans4, uint64_t cap, uint64_t* n_spans);

/* StreamState::flush_buffer's chunk choice (streamer.cpp:29-54) over the n
 * buffered texts: take = head span length unless it is a tail, else max_len. */
int lc_flush_take(const char* const* buffer_texts, uint32_t n, uint32_t structure_aware,
                  uint32_t min_len, uint32_t max_len, uint32_t* take, uint32_t* kind,
                  uint32_t* level);

/* ---- prefill helpers (GPU index build) ---------- */

/* build_index (index.cpp:155-243) for many slots at once on the device from
 * the slots' resident keys.  spans: host [n_spans*4] per slot, concatenated,
 * span_off [n_slots+1]; n_tokens per slot host [n_slots].  Config mirrors
 * IndexConfig (index.hpp:13-22); seeds[slot] = IndexConfig::seed. */
int lc_index_build(lc_index_t h, const uint32_t* n_tokens, const uint32_t* spans,
                   const uint64_t* span_off, double avg_chunks_per_cluster,
                   uint32_t max_coarse_units, uint32_t kmeans_iters, const uint64_t* seeds);

/* Synthetic clustered K/V written straight into the slots: the reference's
 * gen_clustered_workload (workload.cpp:110-169) token stream for seed
 * seeds[slot] (keys/values rounded to bf16 on store), plus texts codes
 * (0 "", 1 "\n") [n_slots*n_tokens] and queries [n_slots*query_count*dim]
 * returned to the host. */
int lc_gen_workload(lc_index_t h, uint32_t n_tokens, uint32_t n_blobs, double concentration,
                    uint32_t query_count, double query_locality, const uint64_t* seeds,
                    uint8_t* text_codes_out, float* queries_out);

#ifdef __cplusplus
}
#endif
#endif /* LYCHEE_B200_H */
