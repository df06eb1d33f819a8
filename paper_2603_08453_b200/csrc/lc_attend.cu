// Gather-based split-K flash-decode over the selected variable-length chunks
// (north star item 3): kernels::attention (kernels.cpp:108-144) for every query
// head of a GQA group at once, over the union of the group's active tokens.
//
// Work partition: a persistent grid (SMs x resident CTAs, 4 warps each).  The
// union active tokens of all slots of the launch form one global sequence
// (slot-major; k_spans wrote each slot's row list and total).  Every warp owns
// an equal contiguous range of that sequence, so the load is balanced to one
// token group no matter how ragged the per-slot selections are, there are no
// waves and no per-CTA prologue per slot.  A warp whose range crosses slot
// boundaries keeps one online-softmax state per slot segment and writes a
// (m, l, o) partial for each; the warp that completes a slot's token count
// merges that slot's partials (log-sum-exp) in warp order (deterministic).
//
// Data movement: each warp streams 16-token groups of gathered K/V rows into a
// private 3-stage shared-memory ring with cp.async (16-byte requests, full
// 128-byte lines; each KV row of the union is read from HBM exactly once).  The
// row ids of a group come from a 4-entry per-warp descriptor ring, loaded four
// groups ahead, so the gather addresses are ready two groups before the copy
// is issued.  The ring is XOR-swizzled so the fragment reads are conflict free.
//
// Math: QK^T and PV on the tensor cores (mma.sync m16n8k16, bf16 in, fp32
// accumulate) with q and the softmax weights split into bf16 hi + lo halves
// (hi in MMA rows 0..G-1, lo in rows 8..8+G-1): products carry ~16 mantissa
// bits over the exact bf16 K/V.  A per-token head mask (row list bits 24..31)
// removes (query, token) pairs outside that head's own active set.
//
// Fragment maps for mma.m16n8k16 (lane = 4r + c):
//   QK: B = K^T, thread (r, c) holds token r (and 8 + r) dims [c*D/4, c*D/4 + D/4),
//       k-step s uses dims c*D/4 + 4s + {0,1,2,3} (a dim permutation applied to
//       both q and k, so the dot product is unchanged).
//   PV: A = P straight from the QK accumulators (FA2 register reuse);
//       B = V, n-tile j <-> dim r*D/8 + j, thread (r, c) holds tokens
//       2c, 2c+1, 8+2c, 9+2c dims [r*D/8, r*D/8 + D/8).
//   Out: thread (r, c) owns query r dims [c*D/4, c*D/4 + D/4).
#include "lc_common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lc {

struct AttendParams {
    Arena a;
    const float* q;  // [slot][G][D]
    float* out;      // [slot][G][D]
    uint32_t n;      // slots of this launch, starting at a.slot0
    float* part;     // [(warps + n)][G][D + 2] per (warp, slot) segment partials
    unsigned long long* prof;  // optional per-warp [t_start, t_stream_end, t_end, groups | smid << 40] (LC_PROF=1)
    uint32_t min_tok;          // head tokens per static warp range, at least (kMinWarpTok)
    PeerGather pg;             // fused all-gather epilogue (pg.n == 0: off)
    AttQueueDev aq;            // streamed mode: tasks published by the selection (k_attend<D, true>)
};

__device__ __forceinline__ unsigned long long gtime_a() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kAttThreads = 128;
constexpr int kAttWarps = kAttThreads / 32;
constexpr int kStages = 3;
constexpr int kRing = 8;   // group descriptors per warp (groups it .. it+5 live)
constexpr int kAhead = 5;  // row lists are fetched this many groups ahead

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void split_bf16(float x, float& hi, float& lo) {
    hi = __bfloat162float(__float2bfloat16_rn(x));
    lo = x - hi;
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(saddr));
    return r;
}

// 16-byte chunk k (0..D/8-1) of staged row `row` -> physical chunk: an XOR
// swizzle that makes both fragment read patterns conflict-free (D = 128)
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t k) {
    return k ^ ((k >> 3) << 1) ^ (row & 7) ^ ((row >> 1) & 1);
}

// first global position of warp w's range
__device__ __forceinline__ uint32_t warp_begin(uint32_t T, uint32_t w, uint32_t NW) {
    return (uint32_t)(((unsigned long long)T * w) / NW);
}
// the warp whose (non-empty) range holds global position pos
__device__ __forceinline__ uint32_t warp_of(uint32_t T, uint32_t pos, uint32_t NW) {
    return (uint32_t)((((unsigned long long)pos + 1) * NW - 1) / T);
}

// Warps that take static ranges: at least kMinWarpTok head tokens each.  A
// launch with few active tokens (one slot, a 32K layer) would otherwise cut
// them into ~1-token ranges over every warp of the persistent grid and leave
// k_merge one partial per warp to combine (measured: 291 us for one slot).
constexpr uint32_t kMinWarpTok = 256;
__device__ __forceinline__ uint32_t active_warps(uint32_t TH, uint32_t NW, uint32_t min_tok) {
    const uint32_t want = (TH + min_tok - 1) / min_tok;
    return want < 1u ? 1u : (want < NW ? want : NW);
}

struct GroupDesc {  // one 16-token group of one slot
    uint32_t slot;  // local slot index, or ~0u when the warp's work is exhausted
    uint32_t pos;   // first token's index in the slot's row list
    uint32_t cnt;   // 1..16
    uint32_t seg;   // partial index of the (range, slot) segment the group belongs to
};

// Work split.  Every slot's union token list is cut into a head (the first 7/8)
// and a tail.  The heads, concatenated, are cut statically into equal
// contiguous warp ranges; the tails, concatenated, form a pool of at most
// kPoolPerWarp x warps chunks that warps claim in order as they finish (SMs
// differ in achieved bandwidth by up to ~30%).  Partial index of a segment:
// static range w of slot s -> w + s, pool chunk k of slot s -> NW + n + k + s
// (both injective because range and slot indices grow together).
constexpr uint32_t kPoolPerWarp = 4;     // pool chunks per warp (upper bound; partial storage)
// Measured on config 2 (round-1 sweep, LC_ATT_* knobs since removed): a 1/8 tail in one chunk per
// warp balances the SMs with the fewest partials (tails 1/2..1/32 and 1..8
// chunks per warp: 156.8 us best vs 166-181 us)
constexpr uint32_t kTailDiv = 8;      // tail = t / kTailDiv of every slot's tokens
constexpr uint32_t kPoolUsed = 1;     // pool chunks per warp actually used (<= kPoolPerWarp)
__device__ __forceinline__ uint32_t head_of(uint32_t t) { return t - t / kTailDiv; }
struct PoolShape {
    uint32_t C;  // pool chunk length (multiple of 16)
    uint32_t K;  // pool chunks
};
__device__ __forceinline__ PoolShape pool_shape(uint32_t TP, uint32_t NW) {
    PoolShape ps;
    const uint32_t kmax = kPoolUsed * NW;
    uint32_t C = (TP + kmax - 1) / kmax;
    C = (C + 15) & ~15u;
    ps.C = C ? C : 16;
    ps.K = (TP + ps.C - 1) / ps.C;
    return ps;
}

// Log-sum-exp combination of head g of slot s from the slot's partials, by one
// warp, in a fixed order (static head ranges wf.., then pool chunks kf..; a
// warp with an empty static range wrote nothing and is skipped): lanes load
// the contributors' (m, l), then every partial row load of a batch is in
// flight at once.
template <int D>
__device__ __forceinline__ void merge_head(float* out, uint32_t* err, uint32_t G, uint32_t g, uint32_t n,
                                           const float* part, uint32_t zero_seg, uint32_t s, uint32_t NW,
                                           uint32_t NWe, uint32_t TH, uint32_t h0, uint32_t h1, uint32_t t0,
                                           uint32_t t1, uint32_t C, const PeerGather& pg, uint32_t slot) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t wf = 1, wl = 0, kf = 1, kl = 0;
    if (h0 < h1) {
        wf = warp_of(TH, h0, NWe);
        wl = warp_of(TH, h1 - 1, NWe);
    }
    if (t0 < t1) {
        kf = t0 / C;
        kl = (t1 - 1) / C;
    }
    const uint32_t nw = wf <= wl ? wl - wf + 1 : 0u, nk = kf <= kl ? kl - kf + 1 : 0u, nc = nw + nk;
    constexpr int PER = D / 32;
    float M = -INFINITY, L = 0.f, o[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) o[k] = 0.f;
    for (uint32_t base = 0; base < nc; base += 32) {
        // lane j of the batch: contributor base + j's row, max and weight
        const uint32_t i = base + lane;
        bool live = false;
        uint32_t seg = zero_seg;
        if (i < nc) {
            if (i < nw) {
                const uint32_t v = wf + i;
                live = warp_begin(TH, v, NWe) < warp_begin(TH, v + 1, NWe);
                seg = v + s;
            } else {
                live = true;
                seg = NW + n + kf + (i - nw) + s;
            }
        }
        const float* ps = part + ((size_t)seg * G + g) * (D + 2);
        const float ms = live ? __ldcg(ps) : -INFINITY;
        const float ls = live ? __ldcg(ps + 1) : 0.f;
        float bm = ms;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
        const float Mn = fmaxf(M, bm);
        if (Mn == -INFINITY) continue;
        const float fo = exp2f(M - Mn);  // rescale what earlier batches accumulated
        L *= fo;
#pragma unroll
        for (int k = 0; k < PER; ++k) o[k] *= fo;
        M = Mn;
        const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
        if (f == 0.f) seg = zero_seg;
        L += f * ls;  // lane-partial, reduced below
        const uint32_t cnt = min(32u, nc - base);
#pragma unroll 8
        for (uint32_t j = 0; j < cnt; ++j) {
            const float fj = __shfl_sync(0xffffffffu, f, j);
            const uint32_t sj = __shfl_sync(0xffffffffu, seg, j);
            const float* pj = part + ((size_t)sj * G + g) * (D + 2) + 2 + lane;
#pragma unroll
            for (int k = 0; k < PER; ++k) o[k] += fj * __ldcg(pj + 32 * k);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
#pragma unroll
    for (int k = 0; k < PER; ++k) out[(size_t)g * D + lane + 32 * k] = L > 0.f ? o[k] / L : 0.f;
    if (!(L > 0.f) && lane == 0) atomicOr(err, kErrEmptyActive);
    if (pg.n) {  // the same row into every rank's gather buffer, then one arrival per rank
        const size_t row = ((size_t)pg.row_of_slot[slot] * G + g) * D;
        for (uint32_t r = 0; r < pg.n; ++r) {
            float* dst = pg.out[r] + row;
#pragma unroll
            for (int k = 0; k < PER; ++k) dst[lane + 32 * k] = L > 0.f ? o[k] / L : 0.f;
        }
        __threadfence_system();
        __syncwarp();
        if (lane == 0)
            for (uint32_t r = 0; r < pg.n; ++r) atomicAdd_system(pg.flag[r], 1u);
    }
}

// One rank's side of the fused all-gather: wait until its arrival counter
// shows `expect` more rows than at the previous wait (the count of waits done
// lives on the device, so the launch replays unchanged in a CUDA graph).
// Bounded: a peer that never writes raises an error bit instead of hanging.
__global__ void k_gather_wait(unsigned int* flag, unsigned int* done, unsigned int expect, uint32_t* err) {
    if (threadIdx.x != 0) return;
    const unsigned int target = (*done + 1u) * expect;
    for (uint32_t spin = 0;; ++spin) {
        unsigned int cur;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(cur) : "l"(flag) : "memory");
        if ((int)(cur - target) >= 0) break;
        if (spin > (1u << 28)) {
            atomicOr(err, kErrGatherTimeout);
            break;
        }
        __nanosleep(64);
    }
    *done += 1u;
}

// Prefix sums of the slots' head / tail token counts (head_of / the rest) over
// the launch's n slots, into shared arrays of n + 1 entries (all threads).
template <int NT>
__device__ __forceinline__ void slot_prefixes(const Arena& a, uint32_t n, uint32_t* s_hp, uint32_t* s_tp,
                                              uint32_t* s_wsum) {
    constexpr int NWP = NT / 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (n + NT - 1) / NT, i0 = tid * per;
    uint32_t lh = 0, lt = 0;
    for (uint32_t i = i0; i < i0 + per && i < n; ++i) {
        const uint32_t t = __ldcg(a.slot_tok + a.slot0 + i);
        lh += head_of(t);
        lt += t - head_of(t);
    }
    uint32_t xh = lh, xt = lt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yh = __shfl_up_sync(0xffffffffu, xh, o), yt = __shfl_up_sync(0xffffffffu, xt, o);
        if (lane >= (uint32_t)o) {
            xh += yh;
            xt += yt;
        }
    }
    if (lane == 31) {
        s_wsum[warp] = xh;
        s_wsum[NWP + warp] = xt;
    }
    __syncthreads();
    uint32_t bh = 0, bt = 0;
    for (uint32_t w = 0; w < warp; ++w) {
        bh += s_wsum[w];
        bt += s_wsum[NWP + w];
    }
    uint32_t rh = bh + xh - lh, rt = bt + xt - lt;
    if (tid == 0) s_hp[0] = s_tp[0] = 0;
    for (uint32_t i = i0; i < i0 + per && i < n; ++i) {
        const uint32_t t = __ldcg(a.slot_tok + a.slot0 + i);
        rh += head_of(t);
        rt += t - head_of(t);
        s_hp[i + 1] = rh;
        s_tp[i + 1] = rt;
    }
    __syncthreads();
}

// After k_attend: one warp per (slot, query head) combines that head's partials
// (log-sum-exp, fixed contributor order -> deterministic); every partial row of
// a batch of contributors is in flight at once.
// Streamed mode: head g of slot s from the partials of the slot's tasks
// [base, base + cnt), in task (= row-list) order -- deterministic.
template <int D>
__device__ __forceinline__ void merge_tasks(float* out, uint32_t* err, uint32_t G, uint32_t g, const float* part,
                                            uint32_t zero_seg, uint32_t base, uint32_t cnt, const PeerGather& pg,
                                            uint32_t slot) {
    const uint32_t lane = threadIdx.x & 31;
    constexpr int PER = D / 32;
    float M = -INFINITY, L = 0.f, o[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) o[k] = 0.f;
    for (uint32_t b0 = 0; b0 < cnt; b0 += 32) {
        const uint32_t i = b0 + lane;
        uint32_t seg = i < cnt ? base + i : zero_seg;
        const float* ps = part + ((size_t)seg * G + g) * (D + 2);
        const float ms = i < cnt ? __ldcg(ps) : -INFINITY;
        const float ls = i < cnt ? __ldcg(ps + 1) : 0.f;
        float bm = ms;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
        const float Mn = fmaxf(M, bm);
        if (Mn == -INFINITY) continue;
        const float fo = exp2f(M - Mn);
        L *= fo;
#pragma unroll
        for (int k = 0; k < PER; ++k) o[k] *= fo;
        M = Mn;
        const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
        if (f == 0.f) seg = zero_seg;
        L += f * ls;
        const uint32_t m = min(32u, cnt - b0);
#pragma unroll 8
        for (uint32_t j = 0; j < m; ++j) {
            const float fj = __shfl_sync(0xffffffffu, f, j);
            const uint32_t sj = __shfl_sync(0xffffffffu, seg, j);
            const float* pj = part + ((size_t)sj * G + g) * (D + 2) + 2 + lane;
#pragma unroll
            for (int k = 0; k < PER; ++k) o[k] += fj * __ldcg(pj + 32 * k);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
#pragma unroll
    for (int k = 0; k < PER; ++k) out[(size_t)g * D + lane + 32 * k] = L > 0.f ? o[k] / L : 0.f;
    if (!(L > 0.f) && lane == 0) atomicOr(err, kErrEmptyActive);
    if (pg.n) {
        const size_t row = ((size_t)pg.row_of_slot[slot] * G + g) * D;
        for (uint32_t r = 0; r < pg.n; ++r) {
            float* dst = pg.out[r] + row;
#pragma unroll
            for (int k = 0; k < PER; ++k) dst[lane + 32 * k] = L > 0.f ? o[k] / L : 0.f;
        }
        __threadfence_system();
        __syncwarp();
        if (lane == 0)
            for (uint32_t r = 0; r < pg.n; ++r) atomicAdd_system(pg.flag[r], 1u);
    }
}

template <int D, bool QUEUE>
__global__ void __launch_bounds__(256) k_merge(AttendParams p, uint32_t NW) {
    const Arena& a = p.a;
    const uint32_t n = p.n, warp = threadIdx.x >> 5, G = a.G;
    if constexpr (QUEUE) {
        pdl_wait();
        const uint32_t x = blockIdx.x * 8 + warp, s = x / G, g = x % G;
        if (s < n)
            merge_tasks<D>(p.out + (size_t)(a.slot0 + s) * G * D, a.err, G, g, p.part + 16,
                           NW + n + kPoolPerWarp * NW + n, __ldcg(p.aq.sbase + s), __ldcg(p.aq.scnt + s), p.pg,
                           a.slot0 + s);
        // the last block out resets the queue and advances the epoch for the next step
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(p.aq.ctl + 4, 1u) == gridDim.x - 1) {
                p.aq.ctl[0] = 0;
                p.aq.ctl[1] = 0;
                p.aq.ctl[2] = 0;
                p.aq.ctl[4] = 0;
                p.aq.ctl[3] = p.aq.ctl[3] + 1u;
                __threadfence();
            }
        }
        return;
    }
    // static partition: the slot totals were final before k_attend started (its
    // own griddepcontrol.wait), so the prefixes need no wait; the partials do
    __shared__ uint32_t s_hp[kMaxAttendSlots + 1], s_tp[kMaxAttendSlots + 1], s_wsum[16];
    slot_prefixes<256>(a, n, s_hp, s_tp, s_wsum);
    pdl_wait();
    const uint32_t x = blockIdx.x * 8 + warp, s = x / G, g = x % G;
    if (s >= n) return;
    if (s_hp[s + 1] == s_hp[s] && s_tp[s + 1] == s_tp[s]) return;  // empty: k_attend wrote zeros
    const uint32_t TH = s_hp[n], TP = s_tp[n];
    const uint32_t NWe = active_warps(TH, NW, p.min_tok);
    const PoolShape pool = pool_shape(TP, NWe);
    merge_head<D>(p.out + (size_t)(a.slot0 + s) * G * D, a.err, G, g, n, p.part + 16, NW + n + kPoolPerWarp * NW + n,
                  s, NW, NWe, TH, s_hp[s], s_hp[s + 1], s_tp[s], s_tp[s + 1], pool.C, p.pg, a.slot0 + s);
}

template <int D, bool QUEUE>
__global__ void __launch_bounds__(kAttThreads, 2) k_attend(AttendParams p) {
    // streamed mode: no grid-wide wait on the selection -- each claimed task is
    // acquired from its publication tag instead
    // (no early griddepcontrol.launch_dependents for k_merge: measured slower,
    // config 2 4217 -> 3994 steps/s with it in the streamed mode)
    if constexpr (!QUEUE) pdl_wait();
    static_assert(D == 64 || D == 128, "D must be 64 or 128");
    constexpr int KS = D / 16;             // k-steps of QK
    constexpr int KW = D / 32;             // 16-byte chunks per thread per K row
    constexpr int NT = D / 8;              // n-tiles of PV
    constexpr int VW = D / 64;             // 16-byte chunks per thread per V row
    constexpr int ROWB = D * 2;            // bytes per K/V row
    constexpr int STAGE = 32 * ROWB;       // 16 K rows + 16 V rows
    const Arena& a = p.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, c = lane & 3;
    const uint32_t G = a.G, n = p.n;

    extern __shared__ __align__(128) unsigned char dsm[];
    unsigned char* ring = dsm + (size_t)warp * kStages * STAGE;  // this warp's stages
    __shared__ uint32_t s_hp[kMaxAttendSlots + 1];  // prefix of the slots' head lengths
    __shared__ uint32_t s_tp[kMaxAttendSlots + 1];  // prefix of the slots' tail lengths
    __shared__ uint32_t s_rows[kAttWarps][kRing][16];
    __shared__ GroupDesc s_gd[kAttWarps][kRing];
    __shared__ uint32_t s_wsum[2 * kAttWarps];

    // ---- prefixes of the slots' head and tail lengths (k_spans wrote the totals) ----
    if constexpr (!QUEUE) slot_prefixes<kAttThreads>(a, n, s_hp, s_tp, s_wsum);
    const uint32_t TH = QUEUE ? 1u : s_hp[n], TP = QUEUE ? 0u : s_tp[n];
    // slots with no active token (reference: sparse_attention throws, retriever.cpp:43)
    if (!QUEUE && blockIdx.x == 0) {
        for (uint32_t s = warp; s < n; s += kAttWarps) {
            if (s_hp[s + 1] != s_hp[s] || s_tp[s + 1] != s_tp[s]) continue;
            for (uint32_t x = lane; x < G * D; x += 32) p.out[(size_t)(a.slot0 + s) * G * D + x] = 0.f;
            if (lane == 0) atomicOr(a.err, kErrEmptyActive);
        }
    }
    const unsigned long long t_start = p.prof ? gtime_a() : 0ull;
    uint32_t n_groups = 0;
    if (TH + TP == 0) return;
    const uint32_t NW = gridDim.x * kAttWarps, w = blockIdx.x * kAttWarps + warp;
    const uint32_t NWe = active_warps(TH, NW, p.min_tok);
    const PoolShape pool = pool_shape(TP, NWe);
    uint32_t* pool_ctr = reinterpret_cast<uint32_t*>(p.part);  // [0] next pool chunk, [1] barrier, [2] CTAs out
    float* part = p.part + 16;

    // ---- group producer: warp-uniform cursor over the static range (positions in
    // the head sequence), then over claimed pool chunks (tail sequence) ----
    auto slot_of = [&](const uint32_t* pre, uint32_t pos) {  // slot holding pos (skips empty ones)
        uint32_t lo = 0, hi = n;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= pos) lo = mid;
            else hi = mid;
        }
        while (pre[lo + 1] <= pos) ++lo;
        return lo;
    };
    const uint32_t* pre = s_hp;  // active sequence: heads, then tails
    bool in_pool = false;
    uint32_t ppos = (!QUEUE && w < NWe) ? warp_begin(TH, w, NWe) : TH;
    uint32_t pend = (!QUEUE && w < NWe) ? warp_begin(TH, w + 1, NWe) : TH;
    uint32_t seg_base = w, ps = (!QUEUE && ppos < pend) ? slot_of(pre, ppos) : 0u;
    // lane 0 claims the next pool chunk one call before the current range runs
    // out (the atomic's latency hides behind one group) -- not earlier, so a
    // slow warp never sits on a chunk a faster one could take
    uint32_t k_next = 0;
    if (!QUEUE && ppos >= pend && lane == 0) k_next = atomicAdd(pool_ctr, 1u);
    bool done = false;
    // streamed mode: the warp's current task (warp-uniform)
    uint32_t q_idx = ~0u, q_pos = 0, q_end = 0, q_slot = 0;
    const uint32_t q_epoch = QUEUE ? __ldcg(p.aq.ctl + 3) : 0u;
    auto claim = [&]() -> bool {  // the next task in publication order; false when none will come
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(p.aq.ctl + 0, 1u);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        for (uint32_t spin = 0;; ++spin) {
            uint32_t tg = ~0u, pub = 0, tail = 0;
            if (lane == 0) {
                if (idx < p.aq.cap)
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(tg) : "l"(p.aq.tag + idx) : "memory");
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(pub) : "l"(p.aq.ctl + 2) : "memory");
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(tail) : "l"(p.aq.ctl + 1) : "memory");
            }
            tg = __shfl_sync(0xffffffffu, tg, 0);
            pub = __shfl_sync(0xffffffffu, pub, 0);
            tail = __shfl_sync(0xffffffffu, tail, 0);
            if (idx < p.aq.cap && tg == q_epoch) break;
            if (pub >= n && idx >= min(tail, p.aq.cap)) return false;
            if (spin > (1u << 26)) {  // bounded: a selection that never publishes raises an error bit
                if (lane == 0) atomicOr(a.err, kErrQueueTimeout);
                return false;
            }
            __nanosleep(128);
        }
        __syncwarp();
        q_idx = idx;
        q_slot = __ldcg(p.aq.t_slot + idx);
        q_pos = __ldcg(p.aq.t_pos + idx);
        q_end = q_pos + __ldcg(p.aq.t_cnt + idx);
        return true;
    };
    auto next_group = [&]() -> GroupDesc {
        GroupDesc gd{~0u, 0u, 0u, 0u};
        if (done) return gd;
        if constexpr (QUEUE) {
            while (q_idx == ~0u || q_pos >= q_end) {
                if (!claim()) {
                    done = true;
                    return gd;
                }
            }
            gd.slot = q_slot;
            gd.pos = q_pos;
            gd.cnt = min(16u, q_end - q_pos);
            gd.seg = q_idx;
            q_pos += gd.cnt;
            return gd;
        }
        if (ppos >= pend) {  // range exhausted: take the claimed pool chunk
            const uint32_t k = __shfl_sync(0xffffffffu, k_next, 0);
            if (k >= pool.K) {
                done = true;
                return gd;
            }
            pre = s_tp;
            in_pool = true;
            ppos = k * pool.C;
            pend = min(TP, ppos + pool.C);
            seg_base = NW + n + k;
            ps = slot_of(pre, ppos);
        }
        const uint32_t se = pre[ps + 1];
        const uint32_t lim = se < pend ? se : pend;
        gd.slot = ps;
        // row-list index: heads first, the tail after the slot's head
        gd.pos = ppos - pre[ps] + (in_pool ? s_hp[ps + 1] - s_hp[ps] : 0u);
        gd.cnt = min(16u, lim - ppos);
        gd.seg = seg_base + ps;
        ppos += gd.cnt;
        if (ppos == se)
            while (ps + 1 < n && pre[ps + 1] <= ppos) ++ps;
        if (ppos >= pend && lane == 0) k_next = atomicAdd(pool_ctr, 1u);
        return gd;
    };
    // descriptor + row entries (row | head mask << 24) of a group into ring entry
    // e: lanes 0..15 cp.async one entry each (padded tokens repeat the last row;
    // the compute masks them by cnt)
    auto fetch = [&](int e) {
        const GroupDesc gd = next_group();
        if (lane == 0) s_gd[warp][e] = gd;
        if (gd.slot != ~0u && lane < 16) {
            const uint32_t* rl = a.rows + (size_t)(a.slot0 + gd.slot) * a.cap_tokens + gd.pos;
            cp_async4((uint32_t)__cvta_generic_to_shared(&s_rows[warp][e][lane]), rl + min((uint32_t)lane, gd.cnt - 1));
        }
    };

    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    // cp.async of one 16-token group into stage `st`: each 8-lane quarter-warp
    // copies one contiguous 128-byte line, so every request is a full line
    auto issue = [&](int e, int st) {
        const GroupDesc gd = s_gd[warp][e];
        if (gd.slot == ~0u) return;
        const unsigned char* Kb = reinterpret_cast<const unsigned char*>(a.K + kv_off(a, a.slot0 + gd.slot));
        const unsigned char* Vb = reinterpret_cast<const unsigned char*>(a.V + kv_off(a, a.slot0 + gd.slot));
        const uint32_t sbase = ring_s + (uint32_t)st * STAGE;
        constexpr int HALVES = ROWB / 128;         // 128-byte segments per row
        constexpr int SEGS = 16 * HALVES;           // segments per 16 rows
#pragma unroll
        for (int e2 = 0; e2 < SEGS / 4; ++e2) {
            const uint32_t id = 4u * e2 + ((uint32_t)lane >> 3);
            const uint32_t row = id / HALVES, half = id % HALVES;
            const uint32_t k = half * 8 + ((uint32_t)lane & 7);  // 16-byte chunk of the row
            const uint32_t src_row = s_rows[warp][e][row] & 0x00ffffffu;
            cp_async16(sbase + row * ROWB + swz(row, k) * 16, Kb + (size_t)src_row * ROWB + k * 16);
            cp_async16(sbase + 16 * ROWB + row * ROWB + swz(row, k) * 16, Vb + (size_t)src_row * ROWB + k * 16);
        }
    };

    // prologue: row lists of groups 0 .. kAhead-1, then two groups in flight
    {
#pragma unroll
        for (int e = 0; e < kAhead; ++e) fetch(e);
        cp_commit();
        cp_wait<0>();
        __syncwarp();
        issue(0, 0);
        cp_commit();
        issue(1, 1);
        cp_commit();
    }

    uint32_t qf[KS][4];
    float acc[NT][4];
    float m_run = -INFINITY, l_run = 0.f;
    uint32_t cur = ~0u, cur_seg = ~0u;
    const float scale = (float)(1.4426950408889634 / sqrt((double)D));

    // partial (m, l, o) of this warp's current segment of slot s; k_merge
    // combines a slot's partials after the kernel (no warp waits on another CTA,
    // so the kernel needs no co-residency guarantee)
    auto flush = [&](uint32_t seg) {
        float l = l_run;
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        if (r < (int)G) {
            float* pr = part + ((size_t)seg * G + r) * (D + 2);
            if (c == 0) {
                pr[0] = m_run;
                pr[1] = l;
            }
            float* o = pr + 2 + c * (D / 4);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                o[j] = acc[j][0] + acc[j][2];
                o[D / 8 + j] = acc[j][1] + acc[j][3];
            }
        }
    };

    for (uint32_t it = 0;; ++it) {
        const int e = (int)(it % kRing);
        const GroupDesc gd = s_gd[warp][e];
        if (gd.slot == ~0u) break;
        ++n_groups;
        // rows of group it + kAhead ride in this iteration's commit group; the
        // K/V of group it + 2 (rows fetched three iterations ago) are issued
        fetch((int)((it + kAhead) % kRing));
        issue((int)((it + 2) % kRing), (int)((it + 2) % kStages));
        cp_commit();
        cp_wait<kStages - 1>();
        __syncwarp();
        if (gd.seg != cur_seg) {
            if (cur_seg != ~0u) flush(cur_seg);
            cur_seg = gd.seg;
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
            m_run = -INFINITY;
            l_run = 0.f;
        }
        if (gd.slot != cur) {
            cur = gd.slot;
            // q fragments: softmax scale and log2(e) folded in, bf16 hi (row r) + lo (row r+8)
            const float* qg = p.q + ((size_t)(a.slot0 + cur) * G + (r < (int)G ? r : 0)) * D + c * (D / 4);
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const float4 qv = __ldg(reinterpret_cast<const float4*>(qg + 4 * s));
                const float qq[4] = {qv.x, qv.y, qv.z, qv.w};
                float h[4], l[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) split_bf16(qq[x] * scale, h[x], l[x]);
                const bool on = r < (int)G;
                qf[s][0] = on ? pack_bf16(h[0], h[1]) : 0u;
                qf[s][2] = on ? pack_bf16(h[2], h[3]) : 0u;
                qf[s][1] = on ? pack_bf16(l[0], l[1]) : 0u;
                qf[s][3] = on ? pack_bf16(l[2], l[3]) : 0u;
            }
        }
        const uint32_t sb = ring_s + (uint32_t)(it % kStages) * STAGE;
        // ---- S = Q K^T (hi rows r, lo rows r+8): even / odd k-steps accumulate
        // separately so the MMA dependency chains are half as long ----
        float sc[2][4], sd[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
            sd[nt][0] = sd[nt][1] = sd[nt][2] = sd[nt][3] = 0.f;
        }
#pragma unroll
        for (int w2 = 0; w2 < KW; ++w2) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const uint32_t row = 8 * nt + r;
                const uint4 kv = lds128(sb + row * ROWB + swz(row, c * KW + w2) * 16);
                mma16816(sc[nt], qf[2 * w2], kv.x, kv.y);
                mma16816(sd[nt], qf[2 * w2 + 1], kv.z, kv.w);
            }
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int x = 0; x < 4; ++x) sc[nt][x] += sd[nt][x];
        // logits of query r for tokens 2c, 2c+1 (nt 0) and 8+2c, 9+2c (nt 1)
        float lg[4];
        bool ok[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int nt = x >> 1, e2 = x & 1;
            lg[x] = sc[nt][e2] + sc[nt][2 + e2];
            const uint32_t tk = nt * 8 + 2 * c + e2;
            ok[x] = r < (int)G && tk < gd.cnt && ((s_rows[warp][e][tk] >> (24 + r)) & 1u);
        }
        float mx = -INFINITY;
#pragma unroll
        for (int x = 0; x < 4; ++x)
            if (ok[x]) mx = fmaxf(mx, lg[x]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run, mx);
        float pr[4];
        float corr = 1.f;
        if (m_new == -INFINITY) {
            pr[0] = pr[1] = pr[2] = pr[3] = 0.f;
        } else {
            corr = exp2f(m_run - m_new);
#pragma unroll
            for (int x = 0; x < 4; ++x) pr[x] = ok[x] ? exp2f(lg[x] - m_new) : 0.f;
            m_run = m_new;
        }
        l_run = l_run * corr + (pr[0] + pr[1]) + (pr[2] + pr[3]);
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                acc[j][0] *= corr;
                acc[j][1] *= corr;
                acc[j][2] *= corr;
                acc[j][3] *= corr;
            }
        }
        // ---- O += P V ----
        uint32_t pa[4];
        {
            float h[4], l[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) split_bf16(pr[x], h[x], l[x]);
            pa[0] = pack_bf16(h[0], h[1]);
            pa[2] = pack_bf16(h[2], h[3]);
            pa[1] = pack_bf16(l[0], l[1]);
            pa[3] = pack_bf16(l[2], l[3]);
        }
        const uint32_t vb = sb + 16 * ROWB;
#pragma unroll
        for (int w2 = 0; w2 < VW; ++w2) {
            uint4 vr[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const uint32_t row = (x >> 1) * 8 + 2 * c + (x & 1);
                vr[x] = lds128(vb + row * ROWB + swz(row, r * VW + w2) * 16);
            }
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int j = w2 * 8 + jj, word = jj >> 1;
                const uint32_t sel = (jj & 1) ? 0x7632u : 0x5410u;
                auto wd = [&](const uint4& u) -> uint32_t {
                    return word == 0 ? u.x : word == 1 ? u.y : word == 2 ? u.z : u.w;
                };
                const uint32_t b0 = __byte_perm(wd(vr[0]), wd(vr[1]), sel);
                const uint32_t b1 = __byte_perm(wd(vr[2]), wd(vr[3]), sel);
                mma16816(acc[j], pa, b0, b1);
            }
        }
        __syncwarp();  // the stage is refilled by a later iteration's issue
    }
    cp_wait<0>();
    if (cur_seg != ~0u) flush(cur_seg);
    const unsigned long long t_merge = p.prof ? gtime_a() : 0ull;

    // the last CTA out resets the pool and the barrier for the next launch
    __syncthreads();
    if (!QUEUE && tid == 0 && atomicAdd(pool_ctr + 2, 1u) == gridDim.x - 1) {
        pool_ctr[0] = 0;
        pool_ctr[1] = 0;
        pool_ctr[2] = 0;
    }
    if (p.prof && lane == 0) {
        unsigned long long* pw = p.prof + (size_t)w * 4;
        pw[0] = t_start;
        pw[1] = t_merge;
        pw[2] = gtime_a();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        pw[3] = n_groups | ((unsigned long long)smid << 40);
    }
}

template <int D>
static constexpr size_t attend_smem() {
    return (size_t)kAttWarps * kStages * 32 * D * 2;
}

template <int D>
static KernelCfg& attend_cfg() {
    static KernelCfg c;
    return c;
}

template <int D, bool QUEUE>
static cudaError_t launch_attend_d(const AttendParams& p, uint32_t grid, cudaStream_t stream,
                                   cudaEvent_t* ev) {
    static KernelCfg qcfg;
    cudaError_t e = QUEUE ? ensure_smem(k_attend<D, true>, qcfg, attend_smem<D>())
                          : ensure_smem(k_attend<D, false>, attend_cfg<D>(), attend_smem<D>());
    if (e != cudaSuccess) return e;
    // lc_attend_timing: an event pair on the launching stream around k_attend
    // alone (k_merge then starts after the second record, without PDL overlap)
    if (ev && (e = cudaEventRecord(ev[0], stream)) != cudaSuccess) return e;
    e = launch_pdl(k_attend<D, QUEUE>, dim3(grid), dim3(kAttThreads), attend_smem<D>(), stream, p);
    if (e != cudaSuccess) return e;
    if (ev && (e = cudaEventRecord(ev[1], stream)) != cudaSuccess) return e;
    return launch_pdl(k_merge<D, QUEUE>, dim3((p.n * p.a.G + 7) / 8), dim3(256), 0, stream, p,
                      grid * (uint32_t)kAttWarps);
}

// Persistent grid: every SM of the current device holds as many CTAs as fit.
uint32_t attend_grid(uint32_t d) {
    return d == 128 ? persistent_grid(k_attend<128, false>, attend_cfg<128>(), kAttThreads, attend_smem<128>())
                    : persistent_grid(k_attend<64, false>, attend_cfg<64>(), kAttThreads, attend_smem<64>());
}

// Task capacity of the streamed mode: every partial row but the zero row
uint32_t attend_queue_cap(uint32_t d, uint32_t G, uint32_t n_slots) {
    const size_t warps = (size_t)attend_grid(d) * kAttWarps, n = std::min<uint32_t>(n_slots, kMaxAttendSlots);
    return (uint32_t)(warps + n + kPoolPerWarp * warps + n);
}

size_t attend_partials_floats(uint32_t d, uint32_t G, uint32_t n_slots) {
    const size_t warps = (size_t)attend_grid(d) * kAttWarps, n = std::min<uint32_t>(n_slots, kMaxAttendSlots);
    return 16 + (warps + n + kPoolPerWarp * warps + n + 1) * G * (d + 2);
}

// Reference-exact mode (fp32 K/V, any head dim): kernels::attention
// (kernels.cpp:108-144) in fp64 -- logits q.k / sqrt(d), max-subtracted
// softmax, weighted value sum -- one warp per query head over the slot's row
// list: per token the lanes split the dims, the logit is a warp sum.
// Reference-exact mode (fp32 K/V): kernels::attention (kernels.cpp:108-144)
// in fp64, split over the row list: CTA (g, slot, z) takes entries
// [z*C, (z+1)*C) of the slot's row list, one token per thread (sequential
// fp64 dot over the fp32 key row), its max, the weights through shared
// memory, and (dim, half) threads accumulating the fp64 value sums; it leaves
// (m, z, o[d]) in fp64.  k_attend_exact_merge combines a head's splits.
__global__ void __launch_bounds__(256) k_attend_exact(Arena a, const float* q, double* part, uint32_t S) {
    const uint32_t g = blockIdx.x, sl = blockIdx.y, zi = blockIdx.z, tid = threadIdx.x;
    const uint32_t slot = a.slot0 + sl, d = a.d, G = a.G;
    const uint32_t n = a.slot_tok[slot];
    const uint32_t C = (n + S - 1) / S, b0 = min(n, zi * C), b1 = min(n, b0 + C);
    const uint32_t* rows = a.rows + (size_t)slot * a.cap_tokens;
    const float* K = a.Kf + kv_off(a, slot);
    const float* V = a.Vf + kv_off(a, slot);
    const float* qg = q + ((size_t)slot * G + g) * d;
    const double scale = 1.0 / sqrt((double)d);
    __shared__ double s_q[256];
    __shared__ double s_w[256], s_acc[256];
    __shared__ uint32_t s_row[256];
    __shared__ double s_mx[8];
    for (uint32_t j = tid; j < d; j += blockDim.x) s_q[j] = (double)qg[j];
    __syncthreads();
    double* pp = part + (((size_t)sl * G + g) * S + zi) * (d + 2);
    // the range's entries in chunks of one per thread: logit, then the chunk max
    double m = -INFINITY, z = 0.0, acc0 = 0.0, acc1 = 0.0;
    const uint32_t j = tid & 127u, h = tid >> 7;
    for (uint32_t base = b0; base < b1; base += blockDim.x) {
        const uint32_t t = base + tid;
        double l = -INFINITY;
        uint32_t row = 0;
        if (t < b1) {
            const uint32_t e = rows[t];
            if ((e >> (24 + g)) & 1u) {
                row = e & 0x00ffffffu;
                const float4* kr = reinterpret_cast<const float4*>(K + (size_t)row * d);
                double s = 0.0;
                for (uint32_t j4 = 0; j4 < d / 4; ++j4) {
                    const float4 kv = __ldg(kr + j4);
                    s = __fma_rn(s_q[4 * j4], (double)kv.x, s);
                    s = __fma_rn(s_q[4 * j4 + 1], (double)kv.y, s);
                    s = __fma_rn(s_q[4 * j4 + 2], (double)kv.z, s);
                    s = __fma_rn(s_q[4 * j4 + 3], (double)kv.w, s);
                }
                l = s * scale;
            }
        }
        double cm = l;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        if ((tid & 31) == 0) s_mx[tid >> 5] = cm;
        __syncthreads();
        cm = -INFINITY;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) cm = fmax(cm, s_mx[w]);
        const double mn = fmax(m, cm);
        if (mn != -INFINITY) {  // rescale what the earlier chunks accumulated
            const double f = m == -INFINITY ? 0.0 : exp(m - mn);
            z *= f;
            acc0 *= f;
            acc1 *= f;
            m = mn;
        }
        s_w[tid] = l == -INFINITY ? 0.0 : exp(l - m);
        s_row[tid] = row;
        __syncthreads();
        const uint32_t cnt = min(blockDim.x, b1 - base), half = (cnt + 1) / 2;
        const uint32_t i0 = h ? half : 0u, i1 = h ? cnt : half;
        for (uint32_t i = i0; i < i1; ++i) {
            const double wi = s_w[i];
            if (wi == 0.0) continue;
            const float* vr = V + (size_t)s_row[i] * d;
            if (j < d) acc0 += wi * (double)vr[j];
            if (j + 128 < d) acc1 += wi * (double)vr[j + 128];
            z += wi;
        }
        __syncthreads();
    }
    if (h == 1) {
        s_acc[j] = acc0;
        s_acc[128 + j] = acc1;
        if (j == 0) s_w[0] = z;
    }
    __syncthreads();
    if (h == 0) {
        if (j < d) pp[2 + j] = acc0 + s_acc[j];
        if (j + 128 < d) pp[2 + j + 128] = acc1 + s_acc[128 + j];
        if (j == 0) {
            pp[0] = m;
            pp[1] = z + s_w[0];
        }
    }
}

__global__ void __launch_bounds__(256) k_attend_exact_merge(Arena a, const double* part, uint32_t S, float* out) {
    const uint32_t g = blockIdx.x, sl = blockIdx.y, tid = threadIdx.x, slot = a.slot0 + sl, d = a.d, G = a.G;
    const double* pp = part + ((size_t)sl * G + g) * S * (d + 2);
    double M = -INFINITY;
    for (uint32_t z = 0; z < S; ++z) M = fmax(M, pp[(size_t)z * (d + 2)]);
    float* og = out + ((size_t)slot * G + g) * d;
    if (M == -INFINITY) {  // sparse_attention over an empty set throws (retriever.cpp:43)
        for (uint32_t j = tid; j < d; j += blockDim.x) og[j] = 0.f;
        if (tid == 0) atomicOr(a.err, kErrEmptyActive);
        return;
    }
    for (uint32_t j = tid; j < d; j += blockDim.x) {
        double num = 0.0, den = 0.0;
        for (uint32_t z = 0; z < S; ++z) {
            const double* pz = pp + (size_t)z * (d + 2);
            if (pz[0] == -INFINITY) continue;
            const double f = exp(pz[0] - M);
            num += f * pz[2 + j];
            den += f * pz[1];
        }
        og[j] = (float)(num / den);
    }
}

// Slots go in launches of at most kMaxAttendSlots whose total token capacity
// fits the kernel's 32-bit global positions.
cudaError_t launch_gather_wait(unsigned int* flag, unsigned int* done, unsigned int expect, uint32_t* err,
                               cudaStream_t stream) {
    k_gather_wait<<<1, 32, 0, stream>>>(flag, done, expect, err);
    return cudaGetLastError();
}

cudaError_t launch_attend(const Arena& a, const float* q, float* out, float* part, uint32_t n_slots,
                          cudaStream_t stream, const PeerGather* pg, const AttQueueDev* aq, cudaEvent_t* att_ev) {
    if (a.kv_f32) {
        // splits per (slot, head): as many as the partials buffer holds, at most 16
        const size_t cap = (attend_partials_floats(a.d, a.G, n_slots) - 16) * 4;
        const size_t per = (size_t)n_slots * a.G * (a.d + 2) * 8;
        const uint32_t S = (uint32_t)std::max<size_t>(1, std::min<size_t>(16, cap / std::max<size_t>(per, 1)));
        double* dp = reinterpret_cast<double*>(part + 16);
        k_attend_exact<<<dim3(a.G, n_slots, S), 256, 0, stream>>>(a, q, dp, S);
        k_attend_exact_merge<<<dim3(a.G, n_slots), 128, 0, stream>>>(a, dp, S, out);
        return cudaGetLastError();
    }
    const uint32_t grid = attend_grid(a.d);
    uint32_t per = kMaxAttendSlots;
    const unsigned long long cap = a.cap_tokens ? a.cap_tokens : 1;
    if ((unsigned long long)per * cap > 0xffffffffull) per = (uint32_t)(0xffffffffull / cap);
    // LC_PROF=1 (diagnostics only): per-warp timestamps, one buffer per device
    static unsigned long long* prof_dev[kMaxDevices] = {};
    const bool want_prof = getenv("LC_PROF") != nullptr;
    unsigned long long*& prof = prof_dev[current_device()];
    if (want_prof && !prof) cudaMalloc(&prof, (size_t)grid * kAttWarps * 4 * 8);
    // streamed: one launch covers every slot of the selection (tasks carry
    // their own positions, so neither the per-launch slot table nor the 32-bit
    // global positions of the static partition apply)
    const bool queued = aq && aq->ctl;
    if (queued) per = n_slots;
    const bool one = n_slots <= per;  // lc_attend_timing times single-launch calls only
    for (uint32_t s0 = 0; s0 < n_slots; s0 += per) {
        AttendParams p{a, q, out, std::min(per, n_slots - s0), part, want_prof ? prof : nullptr, kMinWarpTok,
                       pg ? *pg : PeerGather{nullptr, nullptr, nullptr, 0u}, aq ? *aq : AttQueueDev{}};
        if (const char* ev = getenv("LC_ATT_MINTOK")) p.min_tok = std::max(16, atoi(ev));  // experiments
        if (prof) cudaMemset(prof, 0, (size_t)grid * kAttWarps * 4 * 8);
        p.a.slot0 = a.slot0 + s0;
        cudaError_t e = a.d == 128 ? (queued ? launch_attend_d<128, true>(p, grid, stream, one ? att_ev : nullptr)
                                              : launch_attend_d<128, false>(p, grid, stream, one ? att_ev : nullptr))
                      : a.d == 64  ? (queued ? launch_attend_d<64, true>(p, grid, stream, one ? att_ev : nullptr)
                                              : launch_attend_d<64, false>(p, grid, stream, one ? att_ev : nullptr))
                                   : cudaErrorInvalidValue;
        if (e != cudaSuccess) return e;
        if (want_prof) {
            std::vector<unsigned long long> t((size_t)grid * kAttWarps * 4);
            cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
            unsigned long long t0 = ~0ull, t1 = 0;
            std::vector<double> dur, loopd;
            double pro = 0, grp = 0;
            for (size_t w = 0; w < (size_t)grid * kAttWarps; ++w) {
                const unsigned long long* x = &t[w * 4];
                if (!x[0]) continue;
                t0 = std::min(t0, x[0]);
                t1 = std::max(t1, x[2]);
                dur.push_back((x[2] - x[0]) / 1e3);
                pro += (x[1] - x[0]) / 1e3;
                grp += (double)(x[3] & 0xffffffffull);
            }
            // spread of warp durations inside a CTA vs across SMs
            double in_cta = 0, sm_min = 1e30, sm_max = 0;
            std::vector<double> sm_mean(1024, 0.0), sm_cnt(1024, 0.0);
            for (size_t b = 0; b < grid; ++b) {
                double lo = 1e30, hi = 0;
                for (int k = 0; k < kAttWarps; ++k) {
                    const unsigned long long* x = &t[(b * kAttWarps + k) * 4];
                    if (!x[0]) continue;
                    const double d = (x[2] - x[0]) / 1e3;
                    lo = std::min(lo, d);
                    hi = std::max(hi, d);
                    const uint32_t sm = (uint32_t)(x[3] >> 40) & 1023u;
                    sm_mean[sm] += d;
                    sm_cnt[sm] += 1;
                }
                if (hi > 0) in_cta += hi - lo;
            }
            for (int sm = 0; sm < 1024; ++sm)
                if (sm_cnt[sm] > 0) {
                    sm_min = std::min(sm_min, sm_mean[sm] / sm_cnt[sm]);
                    sm_max = std::max(sm_max, sm_mean[sm] / sm_cnt[sm]);
                }
            fprintf(stderr, "[LC_PROF] k_attend mean in-CTA warp spread %.1f us; per-SM mean warp duration %.1f .. %.1f us\n",
                    in_cta / grid, sm_min, sm_max);
            std::sort(dur.begin(), dur.end());
            if (!dur.empty())
                fprintf(stderr, "[LC_PROF] k_attend warps %zu: dur min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f us | "
                        "stream %.2f us, groups %.1f per warp | first start -> last end %.1f us\n",
                        dur.size(), dur[0], dur[dur.size() / 10], dur[dur.size() / 2], dur[dur.size() * 9 / 10],
                        dur.back(), pro / dur.size(), grp / dur.size(), (t1 - t0) / 1e3);
        }
    }
    return cudaSuccess;
}

}  // namespace lc
