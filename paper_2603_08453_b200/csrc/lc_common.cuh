// Shared device-side definitions for the B200 LycheeCluster decode path.
//
// HBM layout (one arena per engine, slot-major; a slot is one
// (layer, KV head, sequence) single-head engine of the reference):
//
//   K, V        bf16 [slot][cap_tokens][d]           TokenStore keys_/values_ (types.hpp:54-56)
//   chunk_start u32  [slot][cap_chunks+1]            Chunk::span.start; entry M = chunked_end
//   chunk_clu   u32  [slot][cap_chunks]              cluster_of_chunk (internal cluster id)
//   chunk_rep   f32  [slot][cap_chunks][d]           Chunk::rep_key (optional, download only)
//   ucent       f32  [slot][d][cap_units]            CoarseUnit::centroid, dimension-major
//   urad        f64  [slot][cap_units]               CoarseUnit::radius
//   unit_off    u32  [slot][cap_units+1]             CoarseUnit::members as a range of
//                                                    internal fine ids
//   fcent       f32  [slot][cap_clusters][d]         FineCluster::centroid, one row per internal
//                                                    id (the exact fp64 refinement reads a
//                                                    candidate's 512 B row)
//   frow16      f16  [slot][cap_clusters][d]         fcent rounded to nearest fp16, one row per
//                                                    internal id (the certified filters read
//                                                    these; the exact path reads fcent).  The 16 B
//                                                    chunks of a row are XOR-swizzled by the row's
//                                                    position in its unit (swz16): a linear bulk
//                                                    copy of a unit's rows lands in shared memory
//                                                    already conflict-free for the MMA fragments
//   fmeta       u32x4 [slot][cap_clusters]           {radius f64 (lo, hi word), norm bound f32,
//                                                    token_count}: what the filter needs per row,
//                                                    copied next to the rows
//   frad        f64  [slot][cap_clusters]            FineCluster::radius
//   ftok        u32  [slot][cap_clusters]            FineCluster::token_count
//   forig       u32  [slot][cap_clusters]            reference cluster id of internal id
//   fnmem       u32  [slot][cap_clusters]            FineCluster::members.size()
//   funit       u32  [slot][cap_clusters]            FineCluster::parent_unit
//
// Internal fine ids renumber the reference's clusters so that each coarse
// unit's members are contiguous, in the unit's stored (ascending id) order
// (index.cpp:220-241).  All tie-breaks use the reference id (forig).
#pragma once

#include <cstdint>
#include <mutex>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace lc {

constexpr int kMaxGroup = 8;
constexpr uint32_t kMaxAttendSlots = 1024;  // slots per attention launch (global prefix in smem)

struct SlotState {
    uint32_t n_tokens;
    uint32_t chunked_end;
    uint32_t n_chunks;
    uint32_t L;
    uint32_t P;
    uint32_t m0;      // chunks covered by the member CSR (prefill); later ones are grafts
    float rmax;       // upper bound of every fine radius (raised by grafts)
    float cmax;       // upper bound of every fine centroid norm
};

struct Span {  // one contiguous run of active tokens and the query heads it serves
    uint32_t start;
    uint32_t len_mask;  // len << 8 | group mask
};

struct QInfo {  // per query head result summary (mirrors lc_selection_info)
    uint32_t n_units, n_clusters, degenerate, error;
    unsigned long long scanned;
    unsigned long long n_active;
};

// Fused all-gather epilogue: k_merge stores every merged
// (slot, head) output row straight into each rank's gather buffer over
// NVLink peer memory (and the local one), then bumps each rank's arrival
// counter; k_gather_wait releases a rank once its counter shows every row of
// the step.  n == 0: off (outputs go to `out` only).
struct PeerGather {
    float* const* out;            // [n] each rank's gather buffer [rows][G][D] (peer device pointers)
    unsigned int* const* flag;    // [n] each rank's arrival counter
    const uint32_t* row_of_slot;  // [handle slots] gather-buffer row of each slot
    uint32_t n;
};

// Streamed attention work queue (selection -> attention without a grid-wide
// barrier): each selection CTA publishes its slot's row list as tasks of at
// most C tokens once the slot is done; attention warps claim tasks in order
// and wait only for the tasks they claimed.  Tags carry the step's epoch, so
// nothing needs clearing between steps; k_merge's last block resets the
// counters and advances the epoch.  ctl: [0] next task to claim, [1] tasks
// reserved, [2] slots published, [3] epoch, [4] merge blocks out.
struct AttQueueDev {
    uint32_t* ctl;
    uint32_t* t_slot;  // [cap] slot (local to the attention launch)
    uint32_t* t_pos;   // [cap] first row-list entry
    uint32_t* t_cnt;   // [cap] entries
    uint32_t* tag;     // [cap] epoch of the step that published the task
    uint32_t* sbase;   // [n] the slot's first task
    uint32_t* scnt;    // [n] the slot's task count
    uint32_t cap, n;   // task capacity, slots of the launch
    uint32_t cmin;     // minimum tokens per task
};

// One selection CTA's warp publishes its slot's tasks (after every thread's
// row-list writes were fenced and the CTA synchronised): lane 0 reserves the
// task range, the lanes write the tasks, fence, then tag them with the epoch
// (consumers acquire the tag); the published-slot count goes last.
__device__ __forceinline__ void publish_tasks(const AttQueueDev& q, uint32_t lslot, uint32_t tok, uint32_t epoch,
                                              uint32_t* err) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nt_max = q.cap / (q.n ? q.n : 1u) > 0 ? q.cap / (q.n ? q.n : 1u) : 1u;
    uint32_t C = (tok + nt_max - 1) / nt_max;
    C = C < q.cmin ? q.cmin : ((C + 15u) & ~15u);
    const uint32_t nt = tok ? (tok + C - 1) / C : 0u;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(q.ctl + 1, nt);
    base = __shfl_sync(0xffffffffu, base, 0);
    const bool fits = base + nt <= q.cap;
    if (lane == 0) {
        if (!fits) atomicOr(err, 1u << 9);  // kErrQueueOverflow: sized so it cannot happen; the slot's output is then zero
        q.sbase[lslot] = base;
        q.scnt[lslot] = fits ? nt : 0u;
    }
    // every reserved index below the capacity gets a task (empty on overflow),
    // so no attention warp waits on an index that never comes
    const uint32_t lim = base < q.cap ? min(nt, q.cap - base) : 0u;
    for (uint32_t i = lane; i < lim; i += 32) {
        q.t_slot[base + i] = lslot;
        q.t_pos[base + i] = i * C;
        q.t_cnt[base + i] = fits ? min(C, tok - i * C) : 0u;
    }
    __threadfence();
    for (uint32_t i = lane; i < lim; i += 32) *reinterpret_cast<volatile uint32_t*>(q.tag + base + i) = epoch;
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(q.ctl + 2, 1u);
}

struct Arena {
    // shape
    uint32_t n_slots, d, G, cap_tokens, cap_chunks, cap_clusters, cap_units, max_cand;
    uint32_t graft_full, keep_reps, cap_spans;
    uint32_t kv_f32;         // K/V stored as fp32 (Kf, Vf; reference-exact mode) instead of bf16 (K, V)
    uint32_t slot0;          // first slot of the launch (slot groups on several streams)
    // token store
    __nv_bfloat16* K;
    __nv_bfloat16* V;
    float* Kf;
    float* Vf;
    // index
    uint32_t* chunk_start;
    uint32_t* chunk_clu;
    uint32_t* chunk_kl;      // [slot][cap_chunks] kind | level << 8 of chunks grafted on the device
    float* chunk_rep;
    float* ucent;
    double* urad;
    uint32_t* unit_off;
    float* fcent;
    __half* frow16;          // fcent rounded to fp16, one swizzled row per internal id (swz16)
    uint4* fmeta;            // {radius lo, radius hi, norm bound (f32 bits), token_count} per internal id
    double* frad;
    uint32_t* ftok;
    uint32_t* forig;
    uint32_t* fnmem;
    uint32_t* funit;
    uint32_t* fmem_off;      // [slot][cap_clusters+1] member CSR of the prefill chunks (internal ids)
    uint32_t* fmem;          // [slot][cap_chunks] chunk ids, ascending per cluster
    SlotState* state;
    // per-step selection products
    QInfo* qinfo;            // [slot][G]
    uint32_t* sel_units;     // [slot][G][cap_units]
    uint32_t* sel_clusters;  // [slot][G][cap_clusters] reference ids, rank order
    uint32_t* sel_bits;      // [slot][G][words(cap_clusters)] internal-id bitmap
    unsigned char* plan;          // [slot][plan_bytes] coarse-tier plan of the 3-kernel selection
    uint32_t* chunk_bits;         // [slot][G][words(cap_chunks)] per-head active chunk bitmaps
    uint32_t plan_bytes;
    Span* spans;             // [slot][cap_spans]
    uint32_t* span_off;      // [slot][cap_spans+1] token prefix offsets
    uint32_t* n_spans;       // [slot]
    uint32_t* rows;          // [slot][cap_tokens] union active tokens in span order:
                             //   token row | head mask << 24 (k_spans -> k_attend)
    uint32_t* slot_tok;      // [slot] union active token count (length of the row list)
    unsigned long long* step_bytes;  // [slot][4]
    uint32_t* err;           // [1]
};

__host__ __device__ inline uint32_t bit_words(uint32_t n) { return (n + 31) / 32; }

// Per-slot selection plan (k_coarse -> k_fine / k_pickq / k_spans): header
// (256 B), union units u32 [cap_units][4 + G], ucum u32 [cap_units + 1], then
// q as f64 [G][d] at a 16-byte boundary, then the fine tile table
// uint4 [ceil(cap_clusters / 32)] = {first union unit, unit-start bit mask,
// first candidate's index in its unit, 0}.  Returns the total size.
__host__ __device__ inline uint32_t plan_layout(uint32_t cap_units, uint32_t G, uint32_t d, uint32_t cap_clusters,
                                                uint32_t* ucum_off, uint32_t* qd_off, uint32_t* tile_off) {
    const uint32_t u = 256 + cap_units * (4 + G) * 4;
    const uint32_t q = (u + (cap_units + 1) * 4 + 15) & ~15u;
    const uint32_t t = q + G * d * 8;
    if (ucum_off) *ucum_off = u;
    if (qd_off) *qd_off = q;
    if (tile_off) *tile_off = t;
    return t + ((cap_clusters + 31) / 32) * 16;
}

// element (member `local` of the unit block starting at internal id `base`,
// dimension j) of the fine-centroid array: one contiguous 4d-byte row per
// internal id, so the exact refinement of one candidate reads whole lines
__host__ __device__ inline size_t fine_at(uint32_t base, uint32_t nu, uint32_t local, uint32_t j, uint32_t d) {
    (void)nu;
    return ((size_t)base + local) * d + j;
}

// Physical 16-byte chunk of logical chunk k (dims 8k..8k+7) of the fp16 row at
// position `local` of its unit (d = 128: 16 chunks; other head dims are not
// swizzled).  Bits 0-2 of k are XORed with a function of local mod 8 only, so
// rows copied to any shared-memory row with the same residue mod 8 keep the
// pattern: the MMA B-fragment reads (rows r = 0..7, chunks {w, 4+w, 8+w, 12+w})
// then hit 8 distinct bank groups per quarter warp.
__host__ __device__ inline uint32_t swz16(uint32_t local, uint32_t k, uint32_t d) {
    return d == 128 ? (k ^ ((k >> 3) << 1) ^ (local & 7u) ^ ((local >> 1) & 1u)) : k;
}
// element j of internal id (base + local) in the fp16 row array
__host__ __device__ inline size_t frow_at(uint32_t base, uint32_t local, uint32_t j, uint32_t d) {
    return ((size_t)base + local) * d + swz16(local, j >> 3, d) * 8 + (j & 7);
}
// norm bound stored per fine centroid: >= ||c|| of the fp32 centroid
__host__ __device__ inline float norm_bound(double n2) {
    const double n = sqrt(n2) * (1.0 + 1.0 / 1048576.0);
    float f = (float)n;
    if ((double)f < n) f = nextafterf(f, 3.0e38f);
    return f;
}

__host__ __device__ inline size_t kv_off(const Arena& a, uint32_t slot) {
    return (size_t)slot * a.cap_tokens * a.d;
}

// Orderable key of a double so that ascending key == descending score.
__device__ __forceinline__ unsigned long long desc_key(double s) {
    unsigned long long b = (unsigned long long)__double_as_longlong(s);
    unsigned long long ord = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    return ~ord;
}

// Programmatic dependent launch: the kernel may be scheduled while its stream
// predecessor drains; it must run pdl_wait() before touching anything the
// predecessor writes (griddepcontrol.wait returns once the predecessor grid
// has completed and flushed its memory).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- per-device launch configuration (host) --------------------------------
// Device properties, dynamic shared-memory opt-ins and occupancy-derived grid
// sizes are per device: cudaFuncSetAttribute applies to the calling thread's
// current device, so every cache below is keyed by the device ordinal and
// guarded by a mutex (several handles on several devices / threads).
constexpr int kMaxDevices = 64;

struct DevProps {
    int sms = 0, smem_sm = 0, smem_blk = 0;
};

inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev);
}

inline DevProps dev_props() {
    static std::mutex mu;
    static DevProps props[kMaxDevices];
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    DevProps& p = props[dev];
    if (!p.sms) {
        cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&p.smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&p.smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (p.sms <= 0) p.sms = 1;
    }
    return p;
}

// One per kernel instantiation (a function-local static in its launcher).
struct KernelCfg {
    std::mutex mu;
    size_t smem[kMaxDevices] = {};  // dynamic shared memory opted into so far
    uint32_t grid[kMaxDevices] = {};  // persistent grid (SMs x resident CTAs)
    size_t static_smem[kMaxDevices] = {};
    bool have_static[kMaxDevices] = {};
};

// Raise the kernel's dynamic shared-memory limit on the current device to at
// least `need` bytes (only ever raised, so a concurrent smaller request never
// lowers what another launch relies on).  The default limit is 48 KB for
// static + dynamic together, so any dynamic request is opted into explicitly.
template <typename F>
inline cudaError_t ensure_smem(F* func, KernelCfg& c, size_t need) {
    if (need == 0) return cudaSuccess;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(c.mu);
    if (need <= c.smem[dev]) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    if (e == cudaSuccess) c.smem[dev] = need;
    return e;
}

// Persistent grid of the kernel on the current device: SMs x resident CTAs.
template <typename F>
inline uint32_t persistent_grid(F* func, KernelCfg& c, int threads, size_t smem) {
    const int dev = current_device();
    if (ensure_smem(func, c, smem) != cudaSuccess) cudaGetLastError();
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.grid[dev]) {
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, func, threads, smem) != cudaSuccess) cudaGetLastError();
        c.grid[dev] = (uint32_t)dev_props().sms * (uint32_t)(per > 0 ? per : 1);
    }
    return c.grid[dev];
}

template <typename F>
inline size_t static_smem_of(F* func, KernelCfg& c) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.have_static[dev]) {
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, func) != cudaSuccess) cudaGetLastError();
        c.static_smem[dev] = fa.sharedSizeBytes;
        c.have_static[dev] = true;
    }
    return c.static_smem[dev];
}

enum ErrBits : uint32_t {
    kErrNone = 0,
    kErrCandOverflow = 1u << 0,   // fine candidates exceed max_candidates
    kErrEmptyCand = 1u << 1,      // select_topk(k = 0) would throw (retriever.cpp:29)
    kErrSpanOverflow = 1u << 2,   // active spans exceed cap_spans
    kErrZeroNorm = 1u << 3,       // chunk_representative zero norm (index.cpp:36-37)
    kErrChunkCap = 1u << 4,       // graft past cap_chunks
    kErrTokenCap = 1u << 5,       // append past cap_tokens
    kErrEmptyActive = 1u << 6,    // sparse_attention over an empty set (retriever.cpp:43)
    kErrTake = 1u << 7,           // graft take outside the buffered tokens
    kErrGatherTimeout = 1u << 8,  // fused all-gather: a peer's rows never arrived (bounded wait gave up)
    kErrQueueOverflow = 1u << 9,  // streamed attention: task queue full (sized so it cannot happen)
    kErrQueueTimeout = 1u << 10,  // streamed attention: a slot's tasks never published (bounded wait gave up)
};

}  // namespace lc
