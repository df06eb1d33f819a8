// Per-slot fused selection: retrieve_ids() for every query head of a GQA
// group (retriever.cpp:78-159) plus the union active-set construction, in one
// CTA per (layer, KV head, sequence) slot.
//
//   1. coarse tier: the slot's coarse centroids are staged in shared memory
//      once and scored against all G queries (G x P sequential fp64 chains);
//   2. per query: top-k_g units by rank counting (score desc, id asc);
//   3. the UNION of the group's kept units is streamed from HBM exactly once:
//      each warp pulls 32-candidate x 8-quad tiles of the [d/4][n_u][4] unit
//      blocks into a private 3-stage cp.async ring (full 512-byte lines) and
//      runs one sequential DFMA chain per (candidate, query that kept its
//      unit) -- bit-exact kernels::dot, G independent chains per loaded byte;
//   4. per query, on its own warp pair (named barriers): the exact weighted
//      radix select of the token-budget prefix (or fixed k_c) and the rank
//      sort of the selected clusters;
//   5. one pass over the chunk table emits the union of the group's active
//      spans tagged with per-head masks (collect_active, retriever.cpp:60-74).
#include "lc_common.cuh"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lc {

struct SlotSelParams {
    Arena a;
    const float* q;  // [slot][G][d]
    uint32_t unit_topk, mode, cluster_topk, sink, flags;
    unsigned long long budget;
    const uint32_t* buf_off;
    const uint32_t* buf_ids;
    unsigned char* scratch;  // per slot: keys u64 [G][qcap], sel u32 [G][qcap]
    uint32_t qcap;           // per-query candidate capacity of the scratch
    uint32_t pmax;           // max P over slots (shared memory sizing)
    unsigned long long* prof;  // optional phase timestamps [slot][8] (LC_PROF=1)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define LC_MARK(ph) \
    if (p.prof && threadIdx.x == 0) p.prof[(size_t)slot * 8 + (ph)] = gtime();

constexpr int kSSThreads = 256;
constexpr int kSSWarps = kSSThreads / 32;
constexpr int kSSStages = 4;
constexpr int kQuadsPerStage = 4;
constexpr int kStageBytes = kQuadsPerStage * 32 * 16;  // 2 KB
constexpr int kMaxKU = 64;

__device__ __forceinline__ void bar_named(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cpa16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename T>
__device__ __forceinline__ T bscan(T v, T* wt, T& total) {  // block exclusive scan
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T t = lane < kSSWarps ? wt[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kSSWarps) wt[lane] = t;
    }
    __syncthreads();
    const T base = warp > 0 ? wt[warp - 1] : T(0);
    total = wt[kSSWarps - 1];
    __syncthreads();
    return base + x - v;
}

// Dynamic shared memory (all regions 16-byte aligned):
//   qs    f32 [G][D]
//   ukey  u64 [G][pmax]
//   bits  u32 [G][words(cap_clusters)]        per-query selected-cluster bitmaps
//   uu    u32 [pmax][4 + G]                   union units: unit, mask, base, n_u, qoff[G]
//   ring  [warps][stages][4 KB]               fine-tier stages; first the coarse
//                                             staging [D][Pp], last the cluster masks
template <int D, int GQ>
__global__ void __launch_bounds__(kSSThreads, 2) k_select_slot(SlotSelParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Arena& a = p.a;
    const uint32_t slot = a.slot0 + blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t G = GQ;
    constexpr uint32_t d = D, dq = D / 4;
    const SlotState st = a.state[slot];
    const uint32_t n = st.n_tokens, M = st.n_chunks, ce = st.chunked_end, P = st.P, L = st.L;
    const uint32_t all = (1u << G) - 1u;
    QInfo* qi = a.qinfo + (size_t)slot * G;
    Span* sp = a.spans + (size_t)slot * a.cap_spans;
    uint32_t* so = a.span_off + (size_t)slot * (a.cap_spans + 1);
    unsigned long long* sb = a.step_bytes + (size_t)slot * 4;
    const uint32_t wcap = bit_words(a.cap_clusters), words = bit_words(L);

    // degeneracy (retriever.cpp:86-95) is a property of the slot
    if ((p.mode == 1 && (unsigned long long)n <= p.budget) || M == 0) {
        if (tid < G) {
            qi[tid].n_units = P;
            qi[tid].n_clusters = L;
            qi[tid].degenerate = 1;
            qi[tid].error = 0;
            qi[tid].scanned = 0;
            qi[tid].n_active = n;
        }
        if (tid == 0) {
            sp[0].start = 0;
            sp[0].len_mask = (n << 8) | all;
            so[0] = 0;
            so[1] = n;
            a.n_spans[slot] = 1;
            sb[0] = (unsigned long long)d * 4 * n + G * 8ull * d;
            sb[1] = ((unsigned long long)d * 4 * n + 8ull * d) * G;
            sb[2] = n;
            sb[3] = 0;
        }
        return;
    }

    float* qs = reinterpret_cast<float*>(smem);
    unsigned long long* ukey = reinterpret_cast<unsigned long long*>(smem + (size_t)G * D * 4);
    uint32_t* bits = reinterpret_cast<uint32_t*>(ukey + (size_t)G * p.pmax);
    uint32_t* uu = bits + (size_t)G * wcap;
    const uint32_t uu_stride = 4 + G;
    unsigned char* ring = reinterpret_cast<unsigned char*>(uu + (((size_t)p.pmax * uu_stride + 3) & ~3ull));
    const uint32_t Pp = (P + 3) & ~3u;
    float* ucs = reinterpret_cast<float*>(ring);

    __shared__ double s_qnorm[GQ];
    __shared__ uint32_t s_kept[GQ][kMaxKU];
    __shared__ uint32_t s_nu_union, s_nc[GQ], s_ncu;
    __shared__ uint32_t s_gbase[GQ][kMaxKU], s_gpre[GQ][kMaxKU + 1];  // per-query units, ascending
    __shared__ uint32_t hw[GQ][256], hc[GQ][256];
    __shared__ unsigned long long s_kmin[GQ], s_kmax[GQ];
    __shared__ unsigned long long s_prefix[GQ], s_mask[GQ], s_wbefore[GQ];
    __shared__ uint32_t s_cbefore[GQ], s_state[GQ], s_nsel[GQ];
    __shared__ int s_shift[GQ];
    __shared__ unsigned long long wtot[kSSWarps];
    __shared__ uint32_t s_cnt[GQ], s_nsp[GQ];

    LC_MARK(0)
    // ---- phase 0: queries, bitmaps, coarse staging ----
    for (uint32_t x = tid; x < G * D; x += blockDim.x) qs[x] = p.q[(size_t)slot * G * D + x];
    for (uint32_t x = tid; x < G * wcap; x += blockDim.x) bits[x] = 0u;
    if (tid < GQ) {
        s_kmin[tid] = ~0ull;
        s_kmax[tid] = 0ull;
        s_cnt[tid] = 0;
        s_nsp[tid] = 0;
    }
    const float* uc = a.ucent + (size_t)slot * a.cap_units * d;
    {
        const uint32_t pq = Pp >> 2, n4 = D * pq;
        constexpr int kB = 8;
        for (uint32_t e0 = 0; e0 < n4; e0 += kB * kSSThreads) {
            float4 v[kB];
#pragma unroll
            for (int t = 0; t < kB; ++t) {
                const uint32_t e = e0 + t * kSSThreads + tid;
                if (e < n4) v[t] = __ldg(reinterpret_cast<const float4*>(uc + (size_t)(e / pq) * a.cap_units) + e % pq);
            }
#pragma unroll
            for (int t = 0; t < kB; ++t) {
                const uint32_t e = e0 + t * kSSThreads + tid;
                if (e < n4) reinterpret_cast<float4*>(ucs + (size_t)(e / pq) * Pp)[e % pq] = v[t];
            }
        }
    }
    __syncthreads();

    LC_MARK(1)
    // ---- phase 1: ||q_g|| and coarse upper bounds (kernels.cpp:19-23, 155-159) ----
    if (tid < G) {
        double s = 0.0;
        const float* qg = qs + tid * D;
#pragma unroll 8
        for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)qg[j], (double)qg[j], s);
        s_qnorm[tid] = __dsqrt_rn(s);
    }
    const double* ur = a.urad + (size_t)slot * a.cap_units;
    double cdot[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t x = tid + k * kSSThreads;  // (g, u) pair
        double s = 0.0;
        if (x < G * P && tid >= G) {  // threads 0..G-1 are busy with the norms
            const uint32_t g = x / P, u = x % P;
            const float* qg = qs + g * D;
#pragma unroll 8
            for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)qg[j], (double)ucs[j * Pp + u], s);
        }
        cdot[k] = s;
    }
    __syncthreads();
    if (tid < G) {  // the pairs the norm threads skipped
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = tid + k * kSSThreads;
            if (x < G * P) {
                const uint32_t g = x / P, u = x % P;
                const float* qg = qs + g * D;
                double s = 0.0;
                for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)qg[j], (double)ucs[j * Pp + u], s);
                cdot[k] = s;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t x = tid + k * kSSThreads;
        if (x < G * P) {
            const uint32_t g = x / P, u = x % P;
            ukey[(size_t)g * p.pmax + u] = desc_key(__dadd_rn(cdot[k], __dmul_rn(s_qnorm[g], ur[u])));
        }
    }
    __syncthreads();

    // ---- phase 2: per-query top-k_g units (select_topk, retriever.cpp:113-116) ----
    const uint32_t kU = min(min(p.unit_topk, P), (uint32_t)kMaxKU);
    for (uint32_t x = tid; x < G * P; x += blockDim.x) {
        const uint32_t g = x / P, u = x % P;
        const unsigned long long* kg = ukey + (size_t)g * p.pmax;
        const unsigned long long ku = kg[u];
        uint32_t rank = 0;
        for (uint32_t v = 0; v < P; ++v) rank += (kg[v] < ku || (kg[v] == ku && v < u)) ? 1u : 0u;
        if (rank < kU) s_kept[g][rank] = u;
    }
    __syncthreads();
    // ---- phase 3: union of kept units in ascending unit order, per-query offsets ----
    const uint32_t* uoff = a.unit_off + (size_t)slot * (a.cap_units + 1);
    if (warp == 0) {
        // unit masks over P (P <= 1024): lanes own units lane, lane+32, ...
        uint32_t pos = 0;
        uint32_t qacc[GQ];
#pragma unroll
        for (int g = 0; g < GQ; ++g) qacc[g] = 0;
        for (uint32_t u0 = 0; u0 < P; u0 += 32) {
            const uint32_t u = u0 + lane;
            uint32_t m = 0;
            if (u < P)
                for (uint32_t g = 0; g < G; ++g)
                    for (uint32_t k = 0; k < kU; ++k) m |= (s_kept[g][k] == u ? 1u : 0u) << g;
            const unsigned int bal = __ballot_sync(0xffffffffu, m != 0);
            const uint32_t nu = m ? uoff[u + 1] - uoff[u] : 0u;
            // per-query exclusive offsets within this batch of 32 units
            const uint32_t idx = pos + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
            for (uint32_t g = 0; g < G; ++g) {
                const uint32_t mine = ((m >> g) & 1u) ? nu : 0u;
                uint32_t x = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                if (m) uu[idx * uu_stride + 4 + g] = qacc[g] + x - mine;
                qacc[g] += __shfl_sync(0xffffffffu, x, 31);
            }
            if (m) {
                uu[idx * uu_stride + 0] = u;
                uu[idx * uu_stride + 1] = m;
                uu[idx * uu_stride + 2] = uoff[u];
                uu[idx * uu_stride + 3] = nu;
            }
            pos += __popc(bal);
        }
        if (lane == 0) {
            s_nu_union = pos;
            uint32_t acc = 0;
            for (uint32_t k = 0; k < pos; ++k) acc += uu[k * uu_stride + 3];
            s_ncu = acc;
        }
        if (lane < G) s_nc[lane] = qacc[lane];
    }
    __syncthreads();
    if (tid < G) {  // query tid's kept units in ascending unit order (= its candidate order)
        uint32_t k2 = 0;
        for (uint32_t k = 0; k < s_nu_union; ++k)
            if ((uu[k * uu_stride + 1] >> tid) & 1u) {
                s_gbase[tid][k2] = uu[k * uu_stride + 2];
                s_gpre[tid][k2] = uu[k * uu_stride + 4 + tid];
                ++k2;
            }
        s_gpre[tid][k2] = s_nc[tid];
    }
    __syncthreads();
    const uint32_t nuu = s_nu_union, ncu = s_ncu;
    bool overflow = false;
    for (uint32_t g = 0; g < G; ++g) overflow |= s_nc[g] > p.qcap || s_nc[g] == 0;
    if (overflow) {
        if (tid < G) {
            qi[tid].error = s_nc[tid] == 0 ? kErrEmptyCand : kErrCandOverflow;
            qi[tid].degenerate = 0;
            qi[tid].n_units = kU;
            qi[tid].n_clusters = 0;
            qi[tid].scanned = P + s_nc[tid];
            atomicOr(a.err, qi[tid].error);
        }
        return;
    }
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(p.scratch + (size_t)slot * G * p.qcap * 12);
    uint32_t* sel = reinterpret_cast<uint32_t*>(keys + (size_t)G * p.qcap);

    LC_MARK(2)
    // ---- phase 4: fine tier over the union (retriever.cpp:118-135) ----
    const float* fc = a.fcent + (size_t)slot * a.cap_clusters * d;
    const double* fr = a.frad + (size_t)slot * a.cap_clusters;
    const uint32_t* ftk = a.ftok + (size_t)slot * a.cap_clusters;
    {
        const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + warp * kSSStages * kStageBytes;
        const uint32_t ntile = (ncu + 31) / 32;
        const uint32_t my_tiles = ntile > warp ? (ntile - warp + kSSWarps - 1) / kSSWarps : 0u;
        constexpr uint32_t kChunks = dq / kQuadsPerStage;  // stages per 32-candidate tile
        const uint32_t items = my_tiles * kChunks;
        // union candidate ci -> union unit k and its local index (unit sizes in uu)
        auto locate = [&](uint32_t ci, uint32_t& kk) {
            uint32_t k = 0, acc = 0;
            while (k + 1 < nuu && acc + uu[k * uu_stride + 3] <= ci) {
                acc += uu[k * uu_stride + 3];
                ++k;
            }
            kk = k;
            return ci - acc;
        };
        // issue side: the lane's source column for the tile being prefetched
        uint32_t iss_tile = 0xffffffffu, iss_nu = 1;
        const float4* iss_col = nullptr;
        bool iss_ok = false;
        auto issue = [&](uint32_t it) {
            const uint32_t tile = warp + (it / kChunks) * kSSWarps, ch = it % kChunks;
            if (tile != iss_tile) {
                iss_tile = tile;
                const uint32_t ci = tile * 32 + lane;
                iss_ok = ci < ncu;
                if (iss_ok) {
                    uint32_t k;
                    const uint32_t local = locate(ci, k);
                    iss_nu = uu[k * uu_stride + 3];
                    iss_col = reinterpret_cast<const float4*>(fc + (size_t)uu[k * uu_stride + 2] * d) + local;
                }
            }
            const uint32_t stage = ring_s + (it % kSSStages) * kStageBytes;
            if (iss_ok) {
#pragma unroll
                for (int t = 0; t < kQuadsPerStage; ++t)
                    cpa16(stage + t * 512 + lane * 16, iss_col + (size_t)(ch * kQuadsPerStage + t) * iss_nu);
            }
        };
        double chain[GQ];
        uint32_t cm = 0, cloc = 0, ck = 0;
        unsigned long long kmin[GQ], kmax[GQ];
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
            kmin[g] = ~0ull;
            kmax[g] = 0ull;
        }
#pragma unroll
        for (int s = 0; s < kSSStages - 1; ++s) {
            if ((uint32_t)s < items) issue(s);
            cpa_commit();
        }
        for (uint32_t it = 0; it < items; ++it) {
            if (it + kSSStages - 1 < items) issue(it + kSSStages - 1);
            cpa_commit();
            cpa_wait<kSSStages - 1>();
            __syncwarp();
            const uint32_t tile = warp + (it / kChunks) * kSSWarps, ch = it % kChunks;
            if (ch == 0) {
#pragma unroll
                for (int g = 0; g < GQ; ++g) chain[g] = 0.0;
                const uint32_t ci = tile * 32 + lane;
                if (ci < ncu) {
                    cloc = locate(ci, ck);
                    cm = uu[ck * uu_stride + 1];
                } else {
                    cm = 0;
                }
            }
            const unsigned char* stg = ring + (size_t)(warp * kSSStages + it % kSSStages) * kStageBytes;
            if (cm) {
#pragma unroll
                for (int t = 0; t < kQuadsPerStage; ++t) {
                    const float4 v = *reinterpret_cast<const float4*>(stg + t * 512 + lane * 16);
                    const uint32_t jq = ch * kQuadsPerStage + t;
                    const double vx = v.x, vy = v.y, vz = v.z, vw = v.w;
#pragma unroll
                    for (int g = 0; g < GQ; ++g) {
                        if ((cm >> g) & 1u) {
                            const float4 q4 = reinterpret_cast<const float4*>(qs + g * D)[jq];
                            double s = chain[g];
                            s = __fma_rn((double)q4.x, vx, s);
                            s = __fma_rn((double)q4.y, vy, s);
                            s = __fma_rn((double)q4.z, vz, s);
                            s = __fma_rn((double)q4.w, vw, s);
                            chain[g] = s;
                        }
                    }
                }
            }
            __syncwarp();
            if (ch == kChunks - 1 && cm) {
                const uint32_t cid = uu[ck * uu_stride + 2] + cloc;
                const double r = fr[cid];
                const uint32_t w = p.mode == 1 ? ftk[cid] : 1u;
#pragma unroll
                for (int g = 0; g < GQ; ++g) {
                    if ((cm >> g) & 1u) {
                        const unsigned long long key = desc_key(__dadd_rn(chain[g], __dmul_rn(s_qnorm[g], r)));
                        const size_t at = (size_t)g * p.qcap + uu[ck * uu_stride + 4 + g] + cloc;
                        keys[at] = key;
                        sel[at] = w;  // weights live in the selection list until the radix passes end
                        kmin[g] = min(kmin[g], key);
                        kmax[g] = max(kmax[g], key);
                    }
                }
            }
        }
        cpa_wait<0>();
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
            unsigned long long mn = kmin[g], mx = kmax[g];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            if (lane == 0) {
                atomicMin(&s_kmin[g], mn);
                atomicMax(&s_kmax[g], mx);
            }
        }
    }
    __syncthreads();

    LC_MARK(3)
    // ---- phase 5: per-query selection on warp groups (retriever.cpp:140-154) ----
    const uint32_t wpq = G >= kSSWarps ? 1u : (G > 4 ? 1u : (G > 2 ? 2u : (G > 1 ? 4u : 8u)));
    const uint32_t gq = warp / wpq;  // query this warp serves
    const uint32_t nthr = wpq * 32, gt = tid - gq * nthr;
    const uint32_t* fo = a.forig + (size_t)slot * a.cap_clusters;
    const uint32_t* ft = a.ftok + (size_t)slot * a.cap_clusters;
    const unsigned long long budget = p.mode == 1 ? p.budget : (unsigned long long)p.cluster_topk;
    if (gq < G) {
        const uint32_t g = gq, bid = 1 + g, nc = s_nc[g];
        unsigned long long* kg = keys + (size_t)g * p.qcap;
        uint32_t* sg = sel + (size_t)g * p.qcap;
        // candidate index of query g -> internal cluster id
        auto cand = [&](uint32_t i, uint32_t& cid) {
            uint32_t k = 0;
            while (k + 1 < kU && s_gpre[g][k + 1] <= i) ++k;
            cid = s_gbase[g][k] + (i - s_gpre[g][k]);
        };
        if (gt == 0) {
            const unsigned long long mn = s_kmin[g], mx = s_kmax[g];
            const unsigned long long diff = mn ^ mx;
            const int top = diff ? 63 - __clzll((long long)diff) : 0;
            const int shift = (top / 8) * 8;
            const unsigned long long mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
            s_prefix[g] = mn & mask;
            s_mask[g] = mask;
            s_shift[g] = shift;
            s_wbefore[g] = 0;
            s_cbefore[g] = 0;
            s_state[g] = 0;
            s_nsel[g] = 0;
        }
        bar_named(bid, nthr);
        for (int shift = s_shift[g]; shift >= 0; shift -= 8) {
            for (uint32_t b = gt; b < 256; b += nthr) {
                hw[g][b] = 0;
                hc[g][b] = 0;
            }
            bar_named(bid, nthr);
            const unsigned long long prefix = s_prefix[g], mask = s_mask[g];
            for (uint32_t i = gt; i < nc; i += nthr) {
                const unsigned long long k = kg[i];
                if ((k & mask) == prefix) {
                    atomicAdd(&hw[g][(uint32_t)(k >> shift) & 255u], sg[i]);
                    atomicAdd(&hc[g][(uint32_t)(k >> shift) & 255u], 1u);
                }
            }
            bar_named(bid, nthr);
            if (gt < 32) {
                uint32_t w8[8], c8[8];
                unsigned long long lw = 0;
                uint32_t lc = 0;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    w8[t] = hw[g][lane * 8 + t];
                    c8[t] = hc[g][lane * 8 + t];
                    lw += w8[t];
                    lc += c8[t];
                }
                unsigned long long iw = lw;
                uint32_t ic = lc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long yw = __shfl_up_sync(0xffffffffu, iw, o);
                    const uint32_t yc = __shfl_up_sync(0xffffffffu, ic, o);
                    if (lane >= (uint32_t)o) {
                        iw += yw;
                        ic += yc;
                    }
                }
                int found = -1;
                unsigned long long cum = s_wbefore[g] + (iw - lw), wexcl = 0;
                uint32_t ccum = ic - lc, cexcl = 0;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    if (found < 0) {
                        if (cum + w8[t] > budget) {
                            found = t;
                            wexcl = cum;
                            cexcl = ccum;
                        } else {
                            cum += w8[t];
                            ccum += c8[t];
                        }
                    }
                }
                const unsigned int ballot = __ballot_sync(0xffffffffu, found >= 0);
                if (ballot == 0) {
                    if (lane == 0) s_state[g] = 2;
                } else if ((int)lane == __ffs(ballot) - 1) {
                    const uint32_t b = lane * 8 + (uint32_t)found;
                    s_prefix[g] = prefix | ((unsigned long long)b << shift);
                    s_mask[g] = mask | (255ull << shift);
                    s_wbefore[g] = wexcl;
                    s_cbefore[g] += cexcl;
                    s_state[g] = c8[found] == 1 ? 1u : 0u;
                }
            }
            bar_named(bid, nthr);
            if (s_state[g] != 0) break;
        }
        const unsigned long long prefix = s_prefix[g], mask = s_mask[g];
        const uint32_t state = s_state[g], cbefore = s_cbefore[g];
        bar_named(bid, nthr);  // every histogram read of the weights is done
        for (uint32_t base = 0; base < nc; base += nthr) {
            const uint32_t i = base + gt;
            bool take = false;
            if (i < nc) {
                const unsigned long long k = kg[i] & mask;
                take = k < prefix || (k == prefix && (state == 2 || (state == 1 && cbefore == 0)));
            }
            const unsigned int bal = __ballot_sync(0xffffffffu, take);
            uint32_t pos = 0;
            if (lane == 0 && bal) pos = atomicAdd(&s_nsel[g], (uint32_t)__popc(bal));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (take) sg[pos + __popc(bal & ((1u << lane) - 1u))] = i;
        }
        bar_named(bid, nthr);
        if (state == 0 && gt == 0) {  // identical fp64 scores: reference-id order
            unsigned long long used = s_wbefore[g];
            uint32_t admitted = cbefore, last_id = 0;
            bool first = true;
            for (;;) {
                int best = -1;
                uint32_t best_id = 0xffffffffu;
                for (uint32_t i = 0; i < nc; ++i) {
                    if ((kg[i] & mask) != prefix) continue;
                    uint32_t cid;
                    cand(i, cid);
                    const uint32_t oid = fo[cid];
                    if ((first || oid > last_id) && oid < best_id) {
                        best_id = oid;
                        best = (int)i;
                    }
                }
                if (best < 0) break;
                uint32_t cid;
                cand((uint32_t)best, cid);
                const unsigned long long w = p.mode == 1 ? ft[cid] : 1ull;
                if (admitted > 0 && used + w > budget) break;
                used += w;
                ++admitted;
                sg[s_nsel[g]++] = (uint32_t)best;
                last_id = best_id;
                first = false;
            }
        }
        bar_named(bid, nthr);
        const uint32_t nsel = s_nsel[g];
        uint32_t* out_cl = a.sel_clusters + ((size_t)slot * G + g) * a.cap_clusters;
        uint32_t* gbits = bits + (size_t)g * wcap;
        for (uint32_t x = gt; x < nsel; x += nthr) {
            const uint32_t i = sg[x];
            const unsigned long long ki = kg[i];
            uint32_t ci;
            cand(i, ci);
            const uint32_t oi = fo[ci];
            uint32_t rank = 0;
            for (uint32_t y = 0; y < nsel; ++y) {
                const unsigned long long ky = kg[sg[y]];
                if (ky < ki) {
                    ++rank;
                } else if (ky == ki && y != x) {
                    uint32_t cy;
                    cand(sg[y], cy);
                    if (fo[cy] < oi) ++rank;
                }
            }
            out_cl[rank] = oi;
            atomicOr(&gbits[ci >> 5], 1u << (ci & 31));
        }
        uint32_t* out_u = a.sel_units + ((size_t)slot * G + g) * a.cap_units;
        for (uint32_t k = gt; k < kU; k += nthr) out_u[k] = s_kept[g][k];
        if (gt == 0) {
            qi[g].n_units = kU;
            qi[g].n_clusters = nsel;
            qi[g].degenerate = 0;
            qi[g].error = 0;
            qi[g].scanned = (unsigned long long)P + nc;
        }
    }
    __syncthreads();

    LC_MARK(4)
    // ---- phase 6: union active spans (collect_active, retriever.cpp:60-74) ----
    uint8_t* cmask = ring;  // the fine stages are drained
    for (uint32_t c = tid; c < L; c += blockDim.x) {
        uint32_t m = 0;
        for (uint32_t g = 0; g < G; ++g) m |= ((bits[g * wcap + (c >> 5)] >> (c & 31)) & 1u) << g;
        cmask[c] = (uint8_t)m;
    }
    // export the bitmaps (selection download / explicit buffer path)
    uint32_t* gb = a.sel_bits + (size_t)slot * G * wcap;
    for (uint32_t x = tid; x < G * words; x += blockDim.x) gb[(x / words) * wcap + x % words] = bits[(x / words) * wcap + x % words];
    __syncthreads();
    const uint32_t sink_end = min(p.sink, n);
    uint32_t out = 0, tok = 0;
    if (sink_end > 0) {
        if (tid == 0) {
            sp[0].start = 0;
            sp[0].len_mask = (sink_end << 8) | all;
            so[0] = 0;
        }
        out = 1;
        tok = sink_end;
    }
    const uint32_t* cs = a.chunk_start + (size_t)slot * (a.cap_chunks + 1);
    const uint32_t* cc = a.chunk_clu + (size_t)slot * a.cap_chunks;
    uint32_t my_cnt[GQ], my_nsp[GQ];
#pragma unroll
    for (int g = 0; g < GQ; ++g) my_cnt[g] = my_nsp[g] = 0;
    constexpr uint32_t kCPT = 8, kTile = kSSThreads * kCPT;
    for (uint32_t base = 0; base < M; base += kTile) {
        const uint32_t j0 = base + tid * kCPT;
        uint32_t cl[kCPT], m8[kCPT], s8[kCPT], e8[kCPT];
#pragma unroll
        for (int e = 0; e < (int)kCPT; ++e) cl[e] = j0 + e < M ? __ldg(cc + j0 + e) : 0u;
#pragma unroll
        for (int e = 0; e < (int)kCPT; ++e) m8[e] = j0 + e < M ? cmask[cl[e]] : 0u;
#pragma unroll
        for (int e = 0; e < (int)kCPT; ++e) {
            s8[e] = m8[e] ? __ldg(cs + j0 + e) : 0u;
            e8[e] = m8[e] ? __ldg(cs + j0 + e + 1) : 0u;
        }
        uint32_t cnt = 0, toks = 0;
#pragma unroll
        for (int e = 0; e < (int)kCPT; ++e) {
            uint32_t m = m8[e];
            if (m) {
                const uint32_t st0 = max(s8[e], sink_end);
                if (st0 >= e8[e]) {
                    m = 0;
                } else {
                    s8[e] = st0;
                    e8[e] -= st0;  // length
                    cnt += 1;
                    toks += e8[e];
#pragma unroll
                    for (int g = 0; g < GQ; ++g)
                        if ((m >> g) & 1u) {
                            my_cnt[g] += e8[e];
                            my_nsp[g] += 1;
                        }
                }
            }
            m8[e] = m;
        }
        unsigned long long total;
        const unsigned long long ex = bscan<unsigned long long>(((unsigned long long)cnt << 40) | toks, wtot, total);
        uint32_t pos = out + (uint32_t)(ex >> 40), tp = tok + (uint32_t)(ex & 0xffffffffffull);
#pragma unroll
        for (int e = 0; e < (int)kCPT; ++e) {
            if (m8[e]) {
                if (pos < a.cap_spans) {
                    sp[pos].start = s8[e];
                    sp[pos].len_mask = (e8[e] << 8) | m8[e];
                    so[pos] = tp;
                }
                ++pos;
                tp += e8[e];
            }
        }
        out += (uint32_t)(total >> 40);
        tok += (uint32_t)(total & 0xffffffffffull);
    }
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
        const uint32_t c1 = __reduce_add_sync(0xffffffffu, my_cnt[g]);
        const uint32_t c2 = __reduce_add_sync(0xffffffffu, my_nsp[g]);
        if (lane == 0) {
            atomicAdd(&s_cnt[g], c1);
            atomicAdd(&s_nsp[g], c2);
        }
    }
    const uint32_t n_chunk_spans = out - (sink_end > 0 ? 1u : 0u);
    if (p.flags == 1u) {  // buffer_ids = [chunked_end, n), disjoint from the chunks
        const uint32_t b0 = max(ce, sink_end);
        if (n > b0) {
            if (tid == 0 && out < a.cap_spans) {
                sp[out].start = b0;
                sp[out].len_mask = ((n - b0) << 8) | all;
                so[out] = tok;
            }
            ++out;
            tok += n - b0;
        }
    } else if (p.flags == 2u) {  // explicit sorted unique ids
        const uint32_t lo = p.buf_off[slot], hi = p.buf_off[slot + 1];
        for (uint32_t base = lo; base < hi; base += blockDim.x) {
            const uint32_t i = base + tid;
            uint32_t resid = 0, id = 0;
            if (i < hi) {
                id = p.buf_ids[i];
                if (id >= sink_end && id < n) {
                    resid = all;
                    if (id < ce) {  // inside a chunk: drop the heads that already attend it
                        uint32_t l = 0, h = M;
                        while (h - l > 1) {
                            const uint32_t mid = (l + h) >> 1;
                            if (cs[mid] <= id) l = mid;
                            else h = mid;
                        }
                        resid = all & ~(uint32_t)cmask[cc[l]];
                    }
                }
            }
            unsigned long long total;
            const unsigned long long ex = bscan<unsigned long long>(resid ? ((1ull << 40) | 1ull) : 0ull, wtot, total);
            if (resid) {
                const uint32_t pos = out + (uint32_t)(ex >> 40);
                if (pos < a.cap_spans) {
                    sp[pos].start = id;
                    sp[pos].len_mask = (1u << 8) | resid;
                    so[pos] = tok + (uint32_t)(ex & 0xffffffffffull);
                }
                for (uint32_t g = 0; g < G; ++g)
                    if ((resid >> g) & 1u) atomicAdd(&s_cnt[g], 1u);
            }
            out += (uint32_t)(total >> 40);
            tok += (uint32_t)(total & 0xffffffffffull);
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (out > a.cap_spans) {
            atomicOr(a.err, kErrSpanOverflow);
            out = a.cap_spans;
        }
        so[out] = tok;
        a.n_spans[slot] = out;
        const unsigned long long dd = d, Pl = P;
        const uint32_t bufl = (p.flags == 1u && n > max(ce, sink_end)) ? n - max(ce, sink_end) : 0u;
        unsigned long long per_q = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const unsigned long long act = (unsigned long long)s_cnt[g] + sink_end + bufl;
            qi[g].n_active = act;
            per_q += Pl * (4 * dd + 8) + (unsigned long long)s_nc[g] * (4 * dd + 16) +
                     (unsigned long long)s_nsp[g] * 8 + act * 2 * dd * 2 + 8 * dd;
        }
        sb[0] = Pl * (4 * dd + 8) + (unsigned long long)ncu * (4 * dd + 16) + (unsigned long long)n_chunk_spans * 8 +
                (unsigned long long)tok * 2 * dd * 2 + G * 8 * dd;
        sb[1] = per_q;
        sb[2] = tok;
        sb[3] = ncu;
    }
    LC_MARK(5)
}

size_t select_slot_smem_bytes(const Arena& a, uint32_t pmax) {
    const size_t G = a.G;
    size_t b = G * a.d * 4 + G * pmax * 8 + G * bit_words(a.cap_clusters) * 4 +
               (((size_t)pmax * (4 + G) + 3) & ~3ull) * 4;
    size_t ring = (size_t)kSSWarps * kSSStages * kStageBytes;
    const size_t stage_coarse = (size_t)a.d * ((pmax + 3) & ~3u) * 4;
    ring = ring > stage_coarse ? ring : stage_coarse;
    ring = ring > a.cap_clusters ? ring : a.cap_clusters;  // cluster masks reuse the ring
    return b + ring;
}

template <int D, int GQ>
static cudaError_t launch_ss_dg(const SlotSelParams& p, uint32_t n_slots, size_t smem, cudaStream_t stream) {
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(k_select_slot<D, GQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    k_select_slot<D, GQ><<<n_slots, kSSThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_ss_d(const SlotSelParams& p, uint32_t n_slots, size_t smem, cudaStream_t stream) {
    switch (p.a.G) {
        case 1: return launch_ss_dg<D, 1>(p, n_slots, smem, stream);
        case 2: return launch_ss_dg<D, 2>(p, n_slots, smem, stream);
        case 4: return launch_ss_dg<D, 4>(p, n_slots, smem, stream);
        case 8: return launch_ss_dg<D, 8>(p, n_slots, smem, stream);
        default: return cudaErrorInvalidValue;
    }
}

bool select_slot_supports_group(uint32_t g) { return g == 1 || g == 2 || g == 4 || g == 8; }

cudaError_t launch_select_slot(const Arena& a, const float* q, uint32_t unit_topk, uint32_t mode, uint32_t cluster_topk,
                               unsigned long long budget, uint32_t sink, uint32_t flags, const uint32_t* buf_off,
                               const uint32_t* buf_ids, unsigned char* scratch, uint32_t qcap, uint32_t pmax,
                               uint32_t n_slots, cudaStream_t stream) {
    static unsigned long long* prof = nullptr;
    if (getenv("LC_PROF") && !prof) cudaMalloc(&prof, (size_t)a.n_slots * 8 * 8);
    SlotSelParams p{a, q, unit_topk, mode, cluster_topk, sink, flags, budget, buf_off, buf_ids, scratch, qcap, pmax, prof};
    const size_t smem = select_slot_smem_bytes(a, pmax);
    cudaError_t e = a.d == 128 ? launch_ss_d<128>(p, n_slots, smem, stream)
                  : a.d == 64  ? launch_ss_d<64>(p, n_slots, smem, stream)
                               : cudaErrorInvalidValue;
    if (prof && e == cudaSuccess) {  // debug: phase durations averaged over slots
        cudaStreamSynchronize(stream);
        std::vector<unsigned long long> t((size_t)a.n_slots * 8);
        cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
        double acc[5] = {0, 0, 0, 0, 0};
        unsigned long long t0 = ~0ull, t1 = 0;
        for (uint32_t s = a.slot0; s < a.slot0 + n_slots; ++s) {
            for (int k = 0; k < 5; ++k) acc[k] += (double)(t[s * 8 + k + 1] - t[s * 8 + k]);
            t0 = t[s * 8] < t0 ? t[s * 8] : t0;
            t1 = t[s * 8 + 5] > t1 ? t[s * 8 + 5] : t1;
        }
        fprintf(stderr, "[LC_PROF] select_slot per-CTA us: stage %.2f coarse %.2f fine %.2f radix %.2f spans %.2f | span %.1f us\n",
                acc[0] / n_slots / 1e3, acc[1] / n_slots / 1e3, acc[2] / n_slots / 1e3, acc[3] / n_slots / 1e3,
                acc[4] / n_slots / 1e3, (t1 - t0) / 1e3);
    }
    return e;
}

}  // namespace lc
