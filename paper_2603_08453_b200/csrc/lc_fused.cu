// Fused per-slot selection: one CTA per (layer, KV head, sequence) slot runs the
// whole retrieve_ids + collect_active of every query head of its GQA group
// (retriever.cpp:60-154) with no global round trip between the phases:
//
//   P1 coarse   the coarse tier for all G heads (exact sequential fp64 chains,
//               kernels.cpp:155-159), per-head top-k_g units, their union.
//   P2 fine     the union units' fp16 centroid rows stream through a 3-stage
//               shared-memory ring by TMA bulk copies (cp.async.bulk, mbarrier
//               complete_tx; one producer warp, eight consumer warps) and are
//               scored on the tensor cores (mma.sync m16n8k16 f16, q split into
//               fp16 hi + lo rows) as a *certified filter*: every reference
//               upper bound UB = fl64(q.c) + ||q||*r is enclosed in
//               [UB~ - e, UB~ + e].  Each (head, candidate) keeps a 16-bit key:
//               the lower bound quantized (rounded down) on a per-head grid.
//   P3 select   per head on its own warps: weighted radix select of the
//               token-budget prefix on the keys (retriever.cpp:140-154) gives a
//               cut x; the exact fp64 chain (bit-exact kernels::dot) is
//               recomputed only for R = {upper bound >= x}, from the fp32
//               centroids; R is ranked by (score desc, reference id asc) and the
//               prefix walked -- identical to walking the reference's full order
//               (DESIGN.md "certified filter").  Selected clusters' member
//               chunks -> per-head chunk bitmaps in shared memory.
//   P4 spans    union active spans with per-head masks, sink, buffer, the row
//               list k_attend streams (collect_active, retriever.cpp:60-74).
//
// Shapes that do not fit the on-chip capacities (head dim != 128, very long
// contexts) take the four-kernel chain in lc_select3.cu instead.
#include "lc_common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lc {

namespace {

constexpr int kFuThreads = 288;   // 8 consumer warps + 1 producer warp
constexpr int kFuCons = 256;      // threads of the consumer warps
constexpr int kFuD = 128;
constexpr uint32_t kFuRows = 64;  // candidate rows per stage
constexpr uint32_t kFuStages = 3;
constexpr uint32_t kFuStageBytes = kFuRows * kFuD * 2 + kFuRows * 16;  // rows + per-row meta
constexpr uint32_t kFuMaxUnion = 128;
constexpr uint32_t kFuMaxKU = 64;
constexpr uint32_t kFuLC = 256;      // boundary list / R entries per head in shared memory (fast path)
constexpr uint32_t kFuRBytes = 32;   // per entry: exact key, orig, weight, cid, member range, index / rank
constexpr uint32_t kFuColBytes = (kFuD / 4 + 1) * 16;  // one staged fp32 centroid (bank-spread)
constexpr uint32_t kFuSpCache = 1024;

// error-bound constants of the filter: fp16 rounding of c (2^-11),
// q's hi+lo split (2^-22), tensor-core fp32 accumulation over 16 k-steps
// (2^-15, generous), the final hi+lo add (2^-24); subnormal terms 2^-25 sqrt(d)
constexpr double kFuK1 = 5.25e-4;
constexpr double kFuK2 = 3.5e-7;
constexpr double kFuK3 = 5.7e-14;  // 2^-44: the reference's fp64 dot and our fp64 adds

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
// 1D TMA: global -> shared, completion counted on the mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(saddr));
    return r;
}
__device__ __forceinline__ void bar_named(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// inverse of desc_key
__device__ __forceinline__ double key_score64(unsigned long long key) {
    const unsigned long long ord = ~key;
    const unsigned long long b = (ord >> 63) ? (ord & 0x7fffffffffffffffull) : ~ord;
    return __longlong_as_double((long long)b);
}

}  // namespace

struct FusedParams {
    Arena a;
    const float* q;     // [slot][G][D] (k_attend reads it)
    const float* q_in;  // where q is read (host-mapped buffers); copied to q when different
    uint32_t unit_topk, mode, cluster_topk, sink, flags;
    unsigned long long budget;
    const uint32_t* buf_off;
    const uint32_t* buf_ids;
    unsigned char* scratch;  // per slot: keys u64 [G][kc] + u32 [G][kc] (R overflow path)
    uint32_t kc;             // per-head candidate capacity (shared-memory keys)
    uint32_t uc;             // union candidate capacity (shared-memory weights)
    uint32_t smem_a;         // bytes of region A
    uint32_t g8cap;          // entries of the 8-row group table
    uint32_t pf;             // stages requested into L2 beyond the ring
    unsigned long long* prof;  // optional per-slot phase timestamps [slot][8] (LC_PROF=1)
    AttQueueDev aq;            // streamed attention: publish the slot's tasks at the end (aq.ctl null: off)
};

// dynamic shared memory: region A (phase-dependent: coarse tier / stage ring /
// boundary lists and centroid columns / span staging), then the per-head keys,
// chunk bitmaps, first-digit histograms and the 8-row group table
struct FuLayout {
    uint32_t keys, cbits, hist, g8, total;
};
__host__ __device__ inline FuLayout fu_layout(uint32_t smem_a, uint32_t G, uint32_t kc, uint32_t uc, uint32_t mw) {
    FuLayout L;
    uint32_t o = smem_a;
    L.keys = o;
    o += (G * kc * 2 + 15) & ~15u;
    L.cbits = o;
    o += G * mw * 4;
    L.hist = o;
    o += G * 256 * 4;
    L.g8 = o;
    o += ((uc / 8 + kFuMaxUnion + 8) * 4 + 15) & ~15u;
    L.total = o;
    return L;
}
__host__ __device__ inline uint32_t fu_g8cap(uint32_t uc) { return uc / 8 + kFuMaxUnion + 8; }

template <typename T>
__device__ __forceinline__ T fu_scan(T v, T* wt, T& total) {  // exclusive block scan, all threads
    const int nw = (int)(blockDim.x >> 5), lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T t = lane < nw ? wt[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) wt[lane] = t;
    }
    __syncthreads();
    const T base = warp > 0 ? wt[warp - 1] : T(0);
    total = wt[nw - 1];
    __syncthreads();
    return base + x - v;
}

__device__ __forceinline__ unsigned long long fu_time() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define FU_MARK(ph) \
    if (p.prof && threadIdx.x == 0) p.prof[(size_t)(p.a.slot0 + blockIdx.x) * 16 + (ph)] = fu_time();

template <int GQ>
__global__ void __launch_bounds__(kFuThreads, 2) k_select(FusedParams p) {
    pdl_wait();
    // streamed attention: let the attention grid launch as SMs free up; it takes
    // each slot's tasks once this CTA publishes them
    if (p.aq.ctl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t aq_epoch = p.aq.ctl ? __ldcg(p.aq.ctl + 3) : 0u;
    FU_MARK(0)
    constexpr uint32_t G = GQ, D = kFuD;
    constexpr uint32_t GT = kFuCons / GQ;  // threads per head in P3
    const Arena& a = p.a;
    const uint32_t slot = a.slot0 + blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(128) unsigned char sm[];
    const SlotState st = a.state[slot];
    const uint32_t n = st.n_tokens, P = st.P, L = st.L, M = st.n_chunks;
    const uint32_t mwcap = bit_words(a.cap_chunks);
    const FuLayout lay = fu_layout(p.smem_a, G, p.kc, p.uc, mwcap);
    uint16_t* keys = reinterpret_cast<uint16_t*>(sm + lay.keys);      // [G][kc] 16-bit lower-bound keys
    uint32_t* cbits = reinterpret_cast<uint32_t*>(sm + lay.cbits);    // [G][mwcap] active chunks per head
    uint32_t* hist1 = reinterpret_cast<uint32_t*>(sm + lay.hist);     // [G][256] weight by key high byte
    uint32_t* g8 = reinterpret_cast<uint32_t*>(sm + lay.g8);          // 8-row groups of the padded stream
    QInfo* qi = a.qinfo + (size_t)slot * G;

    __shared__ double s_qd[GQ * kFuD];                  // q as f64 (exact chains)
    __shared__ uint32_t s_uu[kFuMaxUnion][4 + GQ];      // union unit: u, mask, base, n_u, per-head offset
    __shared__ uint32_t s_pcum[kFuMaxUnion + 1];        // first row of each union unit in the padded stream
    __shared__ uint16_t s_hk[GQ][kFuMaxKU];             // head's units as union indices (union order)
    __shared__ uint32_t s_nc[GQ];                       // candidates per head
    __shared__ double s_qn[GQ], s_glo[GQ], s_gstep[GQ];
    __shared__ uint32_t s_emax[GQ];
    __shared__ unsigned long long s_bar[2 * kFuStages + 1];  // full[], empty[], coarse tier
    __shared__ uint32_t s_nuu, s_kU, s_ng, s_deg, s_ncu;
    // P3 per head
    __shared__ unsigned long long s_wbefore[GQ];
    __shared__ uint32_t s_b1[GQ], s_kt[GQ], s_ln[GQ], s_nr[GQ], s_nsel[GQ], s_fast[GQ], s_kstar[GQ];
    __shared__ uint32_t s_rbase[GQ + 1];
    __shared__ unsigned long long s_wtot[kFuThreads / 32];

    // ------------------------------------------------------------------ P1
    const bool degenerate = (p.mode == 1 && (unsigned long long)n <= p.budget) || M == 0;
    if (p.q_in != p.q)  // k_attend reads the device copy
        for (uint32_t x = tid; x < G * D; x += kFuThreads)
            const_cast<float*>(p.q)[(size_t)slot * G * D + x] = p.q_in[(size_t)slot * G * D + x];
    if (degenerate) {  // retriever.cpp:86-95: everything, full attention
        const uint32_t all = (1u << G) - 1u;
        Span* sp = a.spans + (size_t)slot * a.cap_spans;
        uint32_t* so = a.span_off + (size_t)slot * (a.cap_spans + 1);
        unsigned long long* sb = a.step_bytes + (size_t)slot * 4;
        const unsigned long long dd = D;
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
            sb[0] = dd * 4 * n + G * 8ull * dd;
            sb[1] = (dd * 4 * n + 8ull * dd) * G;
            sb[2] = n;
            sb[3] = 0;
            a.slot_tok[slot] = n;
        }
        uint32_t* rows = a.rows + (size_t)slot * a.cap_tokens;
        for (uint32_t t = tid; t < n; t += kFuThreads) rows[t] = t | (all << 24);
        if (p.aq.ctl) {
            __threadfence();
            __syncthreads();
            if (warp == 0) publish_tasks(p.aq, blockIdx.x, n, aq_epoch, a.err);
        }
        return;
    }
    const uint32_t CU = a.cap_units;
    {
        // region A: coarse centroids [D][CU] f32 and radii [CU] f64 (TMA), keys [G][P],
        // unit offsets [P + 1], union masks [P]
        float* ucs = reinterpret_cast<float*>(sm);
        double* s_urad = reinterpret_cast<double*>(ucs + (size_t)D * CU);
        unsigned long long* ukey = reinterpret_cast<unsigned long long*>(s_urad + CU);
        uint32_t* s_uoff = reinterpret_cast<uint32_t*>(ukey + (size_t)G * P);
        uint32_t* s_umask = s_uoff + P + 1;
        if (tid == 0) {
            for (uint32_t k = 0; k < 2 * kFuStages + 1; ++k)
                mbar_init(smem_u32(&s_bar[k]), k < kFuStages ? 1u : (k < 2 * kFuStages ? (uint32_t)(kFuCons / 32) : 1u));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            const uint32_t cb = smem_u32(&s_bar[2 * kFuStages]);
            mbar_arrive_tx(cb, D * CU * 4 + CU * 8);
            bulk_g2s(smem_u32(ucs), a.ucent + (size_t)slot * CU * D, D * CU * 4, cb);
            bulk_g2s(smem_u32(s_urad), a.urad + (size_t)slot * CU, CU * 8, cb);
        }
        {  // unit offsets and q in one round of loads
            const uint32_t* uoff = a.unit_off + (size_t)slot * (CU + 1);
            const uint32_t uo = tid <= P ? uoff[tid] : 0u;
            float qv[(kFuD * GQ + kFuThreads - 1) / kFuThreads];
#pragma unroll
            for (int t = 0; t < (int)((kFuD * GQ + kFuThreads - 1) / kFuThreads); ++t) {
                const uint32_t x = tid + t * kFuThreads;
                qv[t] = x < G * D ? p.q_in[(size_t)slot * G * D + x] : 0.f;
            }
            if (tid <= P) s_uoff[tid] = uo;
            if (tid < P) s_umask[tid] = 0;
            for (uint32_t u = tid + kFuThreads; u <= P; u += kFuThreads) {  // P >= kFuThreads
                s_uoff[u] = uoff[u];
                if (u < P) s_umask[u] = 0;
            }
#pragma unroll
            for (int t = 0; t < (int)((kFuD * GQ + kFuThreads - 1) / kFuThreads); ++t) {
                const uint32_t x = tid + t * kFuThreads;
                if (x < G * D) s_qd[x] = (double)qv[t];
            }
        }
        for (uint32_t x = tid; x < G * 256; x += kFuThreads) hist1[x] = 0u;
        if (tid < G) s_emax[tid] = 0u;
        __syncthreads();  // barrier inits, q, offsets
        mbar_wait(smem_u32(&s_bar[2 * kFuStages]), 0);
        FU_MARK(8)
        // ||q_g|| (kernels.cpp:19-23) on the last warp; one thread per unit runs the
        // G coarse dots as independent exact chains
        if (warp == kFuThreads / 32 - 1) {
            if (lane < G) {
                double n2 = 0.0;
#pragma unroll 8
                for (uint32_t j = 0; j < D; ++j) n2 = __fma_rn(s_qd[lane * D + j], s_qd[lane * D + j], n2);
                s_qn[lane] = __dsqrt_rn(n2);
            }
        } else {
            for (uint32_t u = tid; u < P; u += kFuCons) {
                double s[GQ];
#pragma unroll
                for (int g = 0; g < GQ; ++g) s[g] = 0.0;
#pragma unroll 4
                for (uint32_t j = 0; j < D; ++j) {
                    const double c = (double)ucs[j * CU + u];
#pragma unroll
                    for (int g = 0; g < GQ; ++g) s[g] = __fma_rn(s_qd[g * D + j], c, s[g]);
                }
#pragma unroll
                for (int g = 0; g < GQ; ++g) ukey[g * P + u] = __double_as_longlong(s[g]);
            }
        }
        __syncthreads();
        FU_MARK(9)
        for (uint32_t x = tid; x < G * P; x += kFuThreads) {
            const uint32_t g = x / P, u = x % P;
            ukey[x] = desc_key(__dadd_rn(__longlong_as_double(ukey[x]), __dmul_rn(s_qn[g], s_urad[u])));
        }
        __syncthreads();
        const uint32_t kU = min(min(p.unit_topk, P), kFuMaxKU);
        __shared__ uint32_t s_kept[GQ][kFuMaxKU];
        for (uint32_t x = tid; x < G * P; x += kFuThreads) {
            const uint32_t g = x / P, u = x % P;
            const unsigned long long* kg = ukey + (size_t)g * P;
            const unsigned long long ku = kg[u];
            uint32_t rank = 0;
            for (uint32_t v = 0; v < P; ++v) rank += (kg[v] < ku || (kg[v] == ku && v < u)) ? 1u : 0u;
            if (rank < kU) {
                s_kept[g][rank] = u;
                atomicOr(s_umask + u, 1u << g);
            }
        }
        __syncthreads();
        FU_MARK(10)
        for (uint32_t x = tid; x < G * kU; x += kFuThreads)
            a.sel_units[((size_t)slot * G + x / kU) * a.cap_units + x % kU] = s_kept[x / kU][x % kU];
        if (warp == 0) {  // union of the kept units (ascending unit id), per-head offsets, padded rows
            uint32_t pos = 0, npad = 0, ncu = 0;
            uint32_t qacc[GQ], hcnt[GQ];
#pragma unroll
            for (int g = 0; g < GQ; ++g) qacc[g] = hcnt[g] = 0;
            for (uint32_t u0 = 0; u0 < P; u0 += 32) {
                const uint32_t u = u0 + lane;
                uint32_t m = u < P ? s_umask[u] : 0u;
                const uint32_t nu = m ? s_uoff[u + 1] - s_uoff[u] : 0u;
                if (nu == 0) m = 0;  // an empty unit contributes no candidate
                const unsigned int bal = __ballot_sync(0xffffffffu, m != 0);
                const uint32_t idx = pos + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
                for (int g = 0; g < GQ; ++g) {
                    const bool mine = (m >> g) & 1u;
                    const uint32_t cnt = mine ? nu : 0u;
                    uint32_t x = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= (uint32_t)o) x += y;
                    }
                    const unsigned int hb = __ballot_sync(0xffffffffu, mine);
                    if (mine && idx < kFuMaxUnion) {
                        s_uu[idx][4 + g] = qacc[g] + x - cnt;
                        const uint32_t hk = hcnt[g] + __popc(hb & ((1u << lane) - 1u));
                        if (hk < kFuMaxKU) s_hk[g][hk] = (uint16_t)idx;
                    }
                    qacc[g] += __shfl_sync(0xffffffffu, x, 31);
                    hcnt[g] += __popc(hb);
                }
                const uint32_t pad = (nu + 7) & ~7u;
                uint32_t x = pad;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                if (m && idx < kFuMaxUnion) {
                    s_pcum[idx] = npad + x - pad;
                    s_uu[idx][0] = u;
                    s_uu[idx][1] = m;
                    s_uu[idx][2] = s_uoff[u];
                    s_uu[idx][3] = nu;
                }
                npad += __shfl_sync(0xffffffffu, x, 31);
                ncu += __reduce_add_sync(0xffffffffu, nu);
                pos += __popc(bal);
            }
            if (lane == 0) {
                s_nuu = pos;
                s_kU = kU;
                s_ng = npad / 8;
                s_ncu = ncu;
                if (pos <= kFuMaxUnion) s_pcum[pos] = npad;
            }
            if (lane < G) {
                uint32_t nc = 0;
#pragma unroll
                for (int g = 0; g < GQ; ++g)
                    if ((int)lane == g) nc = qacc[g];
                s_nc[lane] = nc;
            }
        }
        __syncthreads();
        if (tid == 0) {
            bool bad = s_nuu > kFuMaxUnion || s_ng > p.g8cap;
            for (uint32_t g = 0; g < G; ++g) bad = bad || s_nc[g] > p.kc || s_nc[g] == 0;
            s_deg = bad ? 1u : 0u;
        }
        if (tid < G) {
            // the head's 16-bit key grid V(q) = lo + q * step: step a power of two and lo a
            // multiple of it, so every V(q) is exact; it spans every possible upper bound
            const double qn = s_qn[tid];
            const double cm = (double)st.cmax, rm = (double)st.rmax;
            const double lo0 = -qn * cm * (1.0 + 1e-6) - 1e-30;
            const double hi0 = qn * (cm + rm) * (1.0 + 1e-6) + 1e-30;
            double step = ldexp(1.0, ilogb((hi0 - lo0) / 65000.0) + 1);
            if (!(step > 0.0) || !(step < 1e300)) step = 1.0;
            s_glo[tid] = floor(lo0 / step) * step;
            s_gstep[tid] = step;
        }
        __syncthreads();
        if (!s_deg) {  // 8-row groups of the padded stream -> (union unit, first local row)
            for (uint32_t k = warp; k < s_nuu; k += kFuThreads / 32) {
                const uint32_t g0 = s_pcum[k] / 8, ng = (s_uu[k][3] + 7) / 8;
                for (uint32_t i = lane; i < ng; i += 32) g8[g0 + i] = (k << 16) | (i * 8);
            }
        }
        __syncthreads();
    }
    if (s_deg) {  // capacity exceeded (the host sizes the capacities from bounds; should not happen)
        if (tid < G) {
            qi[tid].error = s_nc[tid] == 0 ? kErrEmptyCand : kErrCandOverflow;
            qi[tid].degenerate = 0;
            qi[tid].n_units = s_kU;
            qi[tid].n_clusters = 0;
            qi[tid].scanned = (unsigned long long)P + s_nc[tid];
            atomicOr(a.err, qi[tid].error);
        }
        if (tid == 0) {
            a.n_spans[slot] = 0;
            a.span_off[(size_t)slot * (a.cap_spans + 1)] = 0;
            a.slot_tok[slot] = 0;
        }
        if (p.aq.ctl && warp == 0) publish_tasks(p.aq, blockIdx.x, 0u, aq_epoch, a.err);
        return;
    }
    const uint32_t kU = s_kU, ng = s_ng, nstage = (ng + 7) / 8;
    FU_MARK(1)

    // ------------------------------------------------------------------ P2
    const unsigned char* rows_g = reinterpret_cast<const unsigned char*>(a.frow16 + (size_t)slot * a.cap_clusters * D);
    const uint4* meta_g = a.fmeta + (size_t)slot * a.cap_clusters;
    if (warp == kFuThreads / 32 - 1) {
        // producer: stage t holds groups [8t, 8t + 8) of the padded stream; each run of
        // groups of one unit is one bulk copy of its rows (and one of their meta)
        // Warp-parallel: lane j < 8 looks at group 8t + j and, when a run of one unit's
        // groups starts there, issues that run's copies.
        if (lane == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P1 wrote region A
        __syncwarp();
        // one run per lane: (copy source row, rows, stage row); false when no run starts here
        auto run_of = [&](uint32_t t, uint32_t& cid, uint32_t& rows, uint32_t& srow) -> bool {
            const uint32_t gi = 8 * t + lane, ge = min(ng, 8 * t + 8);
            const bool valid = lane < 8 && gi < ge;
            const uint32_t e = valid ? g8[gi] : 0xffffffffu;
            const uint32_t prev = __shfl_up_sync(0xffffffffu, e, 1);
            const bool start = valid && (lane == 0 || (prev >> 16) != (e >> 16));
            const unsigned int sb = __ballot_sync(0xffffffffu, start);
            // the run covers groups [gi, next start or the stage end)
            const unsigned int later = sb & ~((2u << lane) - 1u);
            const uint32_t gend = later ? 8 * t + (__ffs(later) - 1) : ge;
            const uint32_t last = __shfl_sync(0xffffffffu, e, (gend - 8 * t - 1) & 31);
            if (!start) return false;
            const uint32_t k = e >> 16, l0 = e & 0xffffu;
            const uint32_t l1 = min(s_uu[k][3], (last & 0xffffu) + 8);
            cid = s_uu[k][2] + l0;
            rows = l1 - l0;
            srow = 8 * (gi - 8 * t);
            return true;
        };
        // stages beyond the shared-memory ring are requested into L2 ahead of their copy
        auto prefetch = [&](uint32_t t) {
            if (t >= nstage) return;
            uint32_t cid, rows, srow;
            if (run_of(t, cid, rows, srow)) {
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(rows_g + (size_t)cid * D * 2),
                             "r"(rows * D * 2)
                             : "memory");
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(meta_g + cid), "r"(rows * 16)
                             : "memory");
            }
        };
        for (uint32_t t = 0; t < nstage; ++t) {
            const uint32_t s = t % kFuStages;
            if (p.pf) {  // keep stages [t + ring, t + ring + pf) requested into L2
                if (t == 0)
                    for (uint32_t f = kFuStages; f < kFuStages + p.pf; ++f) prefetch(f);
                else
                    prefetch(t + kFuStages + p.pf - 1);
            }
            if (t >= kFuStages) mbar_wait(smem_u32(&s_bar[kFuStages + s]), ((t / kFuStages) - 1) & 1u);
            uint32_t cid = 0, rows = 0, srow = 0;
            const bool mine = run_of(t, cid, rows, srow);
            const uint32_t bytes = __reduce_add_sync(0xffffffffu, mine ? rows * (D * 2 + 16) : 0u);
            const uint32_t fb = smem_u32(&s_bar[s]);
            if (lane == 0) mbar_arrive_tx(fb, bytes);
            __syncwarp();
            if (mine) {
                const uint32_t sbase = smem_u32(sm + s * kFuStageBytes);
                bulk_g2s(sbase + srow * (D * 2), rows_g + (size_t)cid * D * 2, rows * D * 2, fb);
                bulk_g2s(sbase + kFuRows * D * 2 + srow * 16, meta_g + cid, rows * 16, fb);
            }
        }
    } else {
        // consumers: warp w scores the 8 rows of group 8t + w of every stage for all heads
        const uint32_t r = lane >> 2, c = lane & 3;
        uint32_t qf[8][4];
        {
            const uint32_t gr = r < G ? r : 0u;
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const double* qs = s_qd + gr * D + c * 32 + 4 * s;  // exact: q arrived as fp32
                float h[4], lo[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const float qq = (float)qs[x];
                    h[x] = __half2float(__float2half_rn(qq));
                    lo[x] = qq - h[x];
                }
                const bool on = r < G;
                qf[s][0] = on ? pack_h2(h[0], h[1]) : 0u;
                qf[s][2] = on ? pack_h2(h[2], h[3]) : 0u;
                qf[s][1] = on ? pack_h2(lo[0], lo[1]) : 0u;
                qf[s][3] = on ? pack_h2(lo[2], lo[3]) : 0u;
            }
        }
        // epilogue lanes: G <= 4 -> lane row r handles head r & 3, candidate r >> 2 of
        // its column pair; G == 8 -> head r, both candidates
        constexpr uint32_t NJ = GQ > 4 ? 2u : 1u;
        const uint32_t eh = GQ > 4 ? r : (r & 3u);
        const uint32_t ej0 = GQ > 4 ? 0u : (r >> 2);
        const bool ehead = eh < G;
        const double qn = s_qn[ehead ? eh : 0], glo = s_glo[ehead ? eh : 0], gstep = s_gstep[ehead ? eh : 0];
        const double ginv = 1.0 / gstep;
        const double k1 = qn * kFuK1, k2 = qn * kFuK2, k3 = qn * kFuK3;
        uint32_t* hist_h = hist1 + (ehead ? eh : 0) * 256;
        double emax = 0.0;
        for (uint32_t t = 0; t < nstage; ++t) {
            const uint32_t s = t % kFuStages;
            mbar_wait(smem_u32(&s_bar[s]), (t / kFuStages) & 1u);
            const uint32_t gi = 8 * t + warp;
            if (gi < ng) {
                const uint32_t e8 = g8[gi], k = e8 >> 16, l0 = e8 & 0xffffu;
                const uint32_t sb = smem_u32(sm + s * kFuStageBytes);
                float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};
                const uint32_t row = 8 * warp + r;
#pragma unroll
                for (int w2 = 0; w2 < 4; ++w2) {
                    const uint4 kv = lds128(sb + row * (D * 2) + swz16(row, c * 4 + w2, D) * 16);
                    mma_f16(sc, qf[2 * w2], kv.x, kv.y);
                    mma_f16(sd, qf[2 * w2 + 1], kv.z, kv.w);
                }
                float sv[2];
                sv[0] = (sc[0] + sd[0]) + (sc[2] + sd[2]);
                sv[1] = (sc[1] + sd[1]) + (sc[3] + sd[3]);
                if (GQ <= 4) {  // lanes 16..31 take candidate 1 of lane - 16
                    const float o1 = __shfl_up_sync(0xffffffffu, sv[1], 16);
                    if (r >= 4) sv[0] = o1;
                }
                const uint32_t nu = s_uu[k][3], mask = s_uu[k][1], qoff = ehead ? s_uu[k][4 + eh] : 0u;
                const uint4* smeta = reinterpret_cast<const uint4*>(sm + s * kFuStageBytes + kFuRows * D * 2);
#pragma unroll
                for (uint32_t jj = 0; jj < NJ; ++jj) {
                    const uint32_t j = ej0 + jj;
                    const uint32_t rr = 2 * c + j;  // row of the group
                    const uint32_t local = l0 + rr;
                    if (!ehead || local >= nu || !((mask >> eh) & 1u)) continue;
                    const uint4 mt = smeta[8 * warp + rr];
                    const double rad = __hiloint2double((int)mt.y, (int)mt.x);
                    const double cn = (double)__uint_as_float(mt.z);
                    const double ub = __dadd_rn((double)sv[GQ > 4 ? jj : 0], __dmul_rn(qn, rad));
                    const double e = (k1 * cn + k2 + kFuK2 * cn + (fabs(ub) * kFuK3 + k3 * (cn + rad))) * (1.0 + 1e-9) +
                                     1e-300;
                    emax = fmax(emax, e);
                    // q = floor((lb - lo) / step) with the subtraction rounded down: V(q) <= lb
                    // and lb < V(q + 2) (the rounding crosses at most one grid line)
                    const double f = floor(__dsub_rd(__dsub_rd(ub, e), glo) * ginv);
                    const uint32_t q = f <= 0.0 ? 0u : (f >= 65535.0 ? 65535u : (uint32_t)f);
                    const uint32_t key = 65535u - q;
                    keys[eh * p.kc + qoff + local] = (uint16_t)key;
                    atomicAdd(&hist_h[key >> 8], p.mode == 1 ? mt.w : 1u);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s_bar[kFuStages + s]));
        }
        if (ehead) atomicMax(&s_emax[eh], __float_as_uint(__double2float_ru(emax)));
    }
    __syncthreads();
    FU_MARK(2)

    // ------------------------------------------------------------------ P3
    // per head g on GT threads (named barrier 1 + g).  The first radix digit's
    // histogram came with the scores: its boundary bin b1 bounds the cut; the
    // candidates with keys up to bin b1 plus the filter's width form a short list
    // (the walk's prefix, the boundary and every R member); the second digit and R
    // are resolved on that list.
    const uint32_t g = tid / GT, gt = tid % GT;
    const bool in_head = tid < kFuCons;
    const uint32_t hbar = 1 + g;
    unsigned char* rmeta = sm;  // [G][kFuLC] list / R entries (32 B) in region A
    const uint32_t nc = in_head ? s_nc[g] : 0u;
    const unsigned long long budget = p.mode == 1 ? p.budget : (unsigned long long)p.cluster_topk;
    const uint32_t* ftok_g = a.ftok + (size_t)slot * a.cap_clusters;
    const uint32_t* fo = a.forig + (size_t)slot * a.cap_clusters;
    const uint32_t* moff_g = a.fmem_off + (size_t)slot * (a.cap_clusters + 1);
    auto ent = [&](uint32_t h, uint32_t x2) {
        return reinterpret_cast<uint32_t*>(rmeta + ((size_t)h * kFuLC + x2) * kFuRBytes);
    };
    auto cand_of = [&](uint32_t i, uint32_t& k, uint32_t& l) {  // head candidate index -> (union unit, local)
        uint32_t kk = 0;
        while (kk + 1 < kU && s_uu[s_hk[g][kk + 1]][4 + g] <= i) ++kk;
        k = s_hk[g][kk];
        l = i - s_uu[k][4 + g];
    };
    if (in_head) {
        if (gt < 32) {  // first digit: the bin where the weight of the lower-bound order passes the budget
            uint32_t w8[8];
            unsigned long long lw = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                w8[t] = hist1[g * 256 + gt * 8 + t];
                lw += w8[t];
            }
            unsigned long long iw = lw;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, iw, o);
                if (gt >= (uint32_t)o) iw += y;
            }
            int found = -1;
            unsigned long long cum = iw - lw, wexcl = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (found < 0) {
                    if (cum + w8[t] > budget) {
                        found = t;
                        wexcl = cum;
                    } else {
                        cum += w8[t];
                    }
                }
            const unsigned int ballot = __ballot_sync(0xffffffffu, found >= 0);
            if (ballot == 0) {
                if (gt == 0) s_b1[g] = 256u;  // the whole candidate set fits the budget
            } else if ((int)gt == __ffs(ballot) - 1) {
                s_b1[g] = gt * 8 + (uint32_t)found;
                s_wbefore[g] = wexcl;
            }
            if (gt == 0) s_ln[g] = 0;
        }
        bar_named(hbar, GT);
        const uint32_t b1 = s_b1[g];
        // list threshold: every key that can reach R (bin b1's last key + the filter width)
        const double e2 = 2.0 * (double)__uint_as_float(s_emax[g]) * (1.0 + 1e-9);
        const uint32_t dq = (uint32_t)fmin(65535.0, ceil(e2 / s_gstep[g]) + 3.0);
        const uint32_t kt = b1 >= 256 ? 65535u : min(65535u, ((b1 << 8) | 255u) + dq);
        if (gt == 0) s_kt[g] = kt;
        for (uint32_t i0 = 0; i0 < nc; i0 += GT) {
            const uint32_t i = i0 + gt;
            const bool in = i < nc && (b1 >= 256 || keys[g * p.kc + i] <= kt);
            const unsigned int bal = __ballot_sync(0xffffffffu, in);
            uint32_t pos = 0;
            if (lane == 0 && bal) pos = atomicAdd(&s_ln[g], (uint32_t)__popc(bal));
            pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(bal & ((1u << lane) - 1u));
            if (in && pos < kFuLC) ent(g, pos)[7] = i;
        }
        bar_named(hbar, GT);
        const uint32_t ln = s_ln[g];
        if (b1 < 256 && ln <= kFuLC) {
            // list entries: key, weight, cluster, reference id, member range (one round of loads)
            for (uint32_t x2 = gt; x2 < ln; x2 += GT) {
                uint32_t* e = ent(g, x2);
                const uint32_t i = e[7];
                uint32_t k, l;
                cand_of(i, k, l);
                const uint32_t cid = s_uu[k][2] + l;
                e[0] = keys[g * p.kc + i];
                e[2] = fo[cid];
                e[3] = p.mode == 1 ? ftok_g[cid] : 1u;
                e[4] = cid;
                e[5] = moff_g[cid];
                e[6] = moff_g[cid + 1];
            }
            bar_named(hbar, GT);
            if (gt < 32) {  // second digit on the list's bin-b1 entries -> the boundary key K*
                uint32_t* h2 = hist1 + g * 256;
#pragma unroll
                for (int t = 0; t < 8; ++t) h2[gt * 8 + t] = 0u;
                __syncwarp();
                for (uint32_t x2 = gt; x2 < ln; x2 += 32) {
                    const uint32_t* e = ent(g, x2);
                    if ((e[0] >> 8) == b1) atomicAdd(&h2[e[0] & 255u], e[3]);
                }
                __syncwarp();
                uint32_t w8[8];
                unsigned long long lw = 0;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    w8[t] = h2[gt * 8 + t];
                    lw += w8[t];
                }
                unsigned long long iw = lw;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long y = __shfl_up_sync(0xffffffffu, iw, o);
                    if (gt >= (uint32_t)o) iw += y;
                }
                int found = -1;
                unsigned long long cum = s_wbefore[g] + (iw - lw);
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (found < 0) {
                        if (cum + w8[t] > budget) found = t;
                        else cum += w8[t];
                    }
                const unsigned int ballot = __ballot_sync(0xffffffffu, found >= 0);
                const uint32_t b2 = ballot ? __shfl_sync(0xffffffffu, gt * 8 + (uint32_t)max(found, 0), __ffs(ballot) - 1)
                                           : 255u;
                const uint32_t kstar = (b1 << 8) | b2;
                // x = lower edge of K*'s bucket; R = {c : V(q_c + 2) + 2E >= x}, compacted in list order
                const uint32_t qx = 65535u - kstar;
                const double x = qx == 0 ? -INFINITY : s_glo[g] + (double)qx * s_gstep[g];
                uint32_t nr = 0;
                for (uint32_t b = 0; b < ln; b += 32) {
                    const uint32_t x2 = b + gt;
                    uint32_t kq = 0;
                    bool in = false;
                    if (x2 < ln) {
                        kq = ent(g, x2)[0];
                        const uint32_t q0 = 65535u - kq;
                        const double up = q0 + 2 > 65535u ? INFINITY : s_glo[g] + (double)(q0 + 2) * s_gstep[g];
                        in = __dadd_ru(up, e2) >= x;
                    }
                    const unsigned int bal = __ballot_sync(0xffffffffu, in);
                    // move entry x2 to slot nr + rank (slots only move down, read before write)
                    uint32_t v[7];
                    if (in) {
                        const uint32_t* e = ent(g, x2);
#pragma unroll
                        for (int w = 0; w < 7; ++w) v[w] = e[w];
                    }
                    __syncwarp();
                    if (in) {
                        uint32_t* d = ent(g, nr + __popc(bal & ((1u << gt) - 1u)));
#pragma unroll
                        for (int w = 0; w < 7; ++w) d[w] = v[w];
                    }
                    __syncwarp();
                    nr += __popc(bal);
                }
                if (gt == 0) {
                    s_nr[g] = nr;
                    s_kstar[g] = kstar;
                    s_fast[g] = 1;
                }
            }
        } else if (gt == 0) {
            s_fast[g] = 0;  // everything fits the budget, or the list overflowed: general path
            s_nr[g] = 0;
        }
    }
    __syncthreads();
    FU_MARK(11)
    // R of every fast head, concatenated in head order: exact fp64 chains (bit-exact
    // kernels::dot) from the fp32 centroid rows, staged by cp.async into column slots in
    // region A's tail and the (now dead) key region
    if (tid == 0) {
        uint32_t acc = 0;
        for (uint32_t h = 0; h < G; ++h) {
            s_rbase[h] = acc;
            acc += s_fast[h] ? s_nr[h] : 0u;
        }
        s_rbase[G] = acc;
    }
    __syncthreads();
    FU_MARK(12)
    {
        const uint32_t ntot = s_rbase[G];
        const uint32_t a_used = G * kFuLC * kFuRBytes;
        const uint32_t na = (p.smem_a - a_used) / kFuColBytes;
        bool any_slow = false;
        for (uint32_t h = 0; h < G; ++h) any_slow = any_slow || !s_fast[h];
        // a slow head still reads its keys after this
        const uint32_t nk = any_slow ? 0u : (lay.cbits - lay.keys) / kFuColBytes;
        const uint32_t nslots = na + nk;
        const float* fcs = a.fcent + (size_t)slot * a.cap_clusters * D;
        auto col = [&](uint32_t k) -> unsigned char* {
            return k < na ? sm + a_used + (size_t)k * kFuColBytes : sm + lay.keys + (size_t)(k - na) * kFuColBytes;
        };
        auto rent = [&](uint32_t x2, uint32_t& h) -> uint32_t* {  // R entry x2 of the concatenation
            h = 0;
            while (h + 1 < G && s_rbase[h + 1] <= x2) ++h;
            return ent(h, x2 - s_rbase[h]);
        };
        for (uint32_t r0 = 0; r0 < ntot; r0 += nslots) {
            const uint32_t cnt = min(nslots, ntot - r0);
            for (uint32_t x2 = tid; x2 < cnt * (D / 4); x2 += kFuThreads) {
                uint32_t h;
                const uint32_t* e = rent(r0 + x2 / (D / 4), h);
                const float4* src = reinterpret_cast<const float4*>(fcs + (size_t)e[4] * D) + x2 % (D / 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                                 smem_u32(col(x2 / (D / 4)) + (x2 % (D / 4)) * 16)),
                             "l"(src));
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            __syncthreads();
            for (uint32_t t = tid; t < cnt; t += kFuThreads) {
                uint32_t h;
                uint32_t* e = rent(r0 + t, h);
                const float4* cv = reinterpret_cast<const float4*>(col(t));
                // the radius load is issued before the dot chain, so its latency overlaps it
                const double rad = __ldg(a.frad + (size_t)slot * a.cap_clusters + e[4]);
                double sacc = 0.0;
#pragma unroll 8
                for (uint32_t jq = 0; jq < D / 4; ++jq) {
                    const float4 v = cv[jq];
                    sacc = __fma_rn(s_qd[h * D + 4 * jq + 0], (double)v.x, sacc);
                    sacc = __fma_rn(s_qd[h * D + 4 * jq + 1], (double)v.y, sacc);
                    sacc = __fma_rn(s_qd[h * D + 4 * jq + 2], (double)v.z, sacc);
                    sacc = __fma_rn(s_qd[h * D + 4 * jq + 3], (double)v.w, sacc);
                }
                const unsigned long long kx = desc_key(__dadd_rn(sacc, __dmul_rn(s_qn[h], rad)));
                e[0] = (uint32_t)kx;
                e[1] = (uint32_t)(kx >> 32);
            }
            __syncthreads();
        }
    }
    FU_MARK(3)
    // rank R by (exact key asc, reference id asc) = select_topk's order, walk the prefix
    uint32_t* out_cl = a.sel_clusters + ((size_t)slot * G + (in_head ? g : 0)) * a.cap_clusters;
    uint32_t* cb = cbits + (size_t)(in_head ? g : 0) * mwcap;
    const bool grafted = st.m0 < M;
    uint32_t* clb = a.sel_bits + ((size_t)slot * G + (in_head ? g : 0)) * bit_words(a.cap_clusters);
    if (in_head) {
        for (uint32_t w = gt; w < bit_words(M); w += GT) cb[w] = 0u;
        if (grafted)
            for (uint32_t w = gt; w < bit_words(L); w += GT) clb[w] = 0u;
    }
    const uint32_t* mem = a.fmem + (size_t)slot * a.cap_chunks;
    const uint32_t* cs_g = a.chunk_start + (size_t)slot * (a.cap_chunks + 1);
    if (in_head && s_fast[g]) {
        bar_named(hbar, GT);  // bitmaps cleared
        const uint32_t nr = s_nr[g];
        for (uint32_t x2 = gt; x2 < nr; x2 += GT) {
            const uint32_t* e = ent(g, x2);
            const unsigned long long kr = ((unsigned long long)e[1] << 32) | e[0];
            const uint32_t orr = e[2];
            uint32_t rank = 0;
            for (uint32_t y = 0; y < nr; ++y) {
                const uint32_t* f = ent(g, y);
                const unsigned long long ky = ((unsigned long long)f[1] << 32) | f[0];
                rank += (ky < kr || (ky == kr && f[2] < orr)) ? 1u : 0u;
            }
            ent(g, rank)[7] = x2;  // rank -> entry (word 7 is free again)
        }
        bar_named(hbar, GT);
        if (gt < 32) {  // running weight; the first overflow ends the prefix (first admitted always)
            unsigned long long run = 0;
            uint32_t nsel = nr;
            for (uint32_t b = 0; b < nr; b += 32) {
                const uint32_t rr = b + gt;
                unsigned long long x2 = rr < nr ? (unsigned long long)ent(g, ent(g, rr)[7])[3] : 0ull;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long y = __shfl_up_sync(0xffffffffu, x2, o);
                    if (gt >= (uint32_t)o) x2 += y;
                }
                const bool over = rr < nr && rr > 0 && run + x2 > budget;
                const unsigned int bal = __ballot_sync(0xffffffffu, over);
                if (bal) {
                    nsel = b + __ffs(bal) - 1;
                    break;
                }
                run += __shfl_sync(0xffffffffu, x2, 31);
            }
            if (gt == 0) s_nsel[g] = nsel;
        }
        bar_named(hbar, GT);
        // selected clusters in rank order; member chunks over the lanes of a warp (their
        // span bounds prefetched into L2 for the span phase)
        // One lane per selected cluster (the warp's clusters x2 = hw_ + k * GT/32),
        // so every cluster's member-list loads are in flight together instead
        // of one dependent round trip per cluster; clusters with long member
        // lists (grafted runs) go over the warp's lanes afterwards.
        const uint32_t nsel = s_nsel[g], hw_ = gt >> 5;
        constexpr uint32_t kLaneMembers = 8;
        for (uint32_t base = hw_; base < nsel; base += 32 * (GT / 32)) {
            const uint32_t x2 = base + lane * (GT / 32);
            const uint32_t* e = x2 < nsel ? ent(g, ent(g, x2)[7]) : nullptr;
            bool longl = false;
            if (e) {
                out_cl[x2] = e[2];
                if (grafted) atomicOr(&clb[e[4] >> 5], 1u << (e[4] & 31));
                const uint32_t t0 = e[5], t1 = e[6];
                longl = t1 - t0 > kLaneMembers;
                if (!longl) {
                    uint32_t j[kLaneMembers];
#pragma unroll
                    for (uint32_t k = 0; k < kLaneMembers; ++k)
                        if (t0 + k < t1) j[k] = mem[t0 + k];
#pragma unroll
                    for (uint32_t k = 0; k < kLaneMembers; ++k)
                        if (t0 + k < t1) {
                            atomicOr(&cb[j[k] >> 5], 1u << (j[k] & 31));
                            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(cs_g + j[k]));
                        }
                }
            }
            for (unsigned int lb = __ballot_sync(0xffffffffu, longl); lb; lb &= lb - 1u) {
                const uint32_t* el = ent(g, ent(g, base + (uint32_t)(__ffs(lb) - 1) * (GT / 32))[7]);
                for (uint32_t t = el[5] + lane; t < el[6]; t += 32) {
                    const uint32_t jj = mem[t];
                    atomicOr(&cb[jj >> 5], 1u << (jj & 31));
                    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(cs_g + jj));
                }
            }
        }
    } else if (in_head) {
        // the whole candidate set fits the budget, or a long list: exact keys for every
        // candidate that can reach R in global scratch, an exact radix select, the rank
        // of the selection (k_pickq's general path)
        unsigned long long* kg = reinterpret_cast<unsigned long long*>(p.scratch + (size_t)slot * G * p.kc * 12) +
                                 (size_t)g * p.kc;
        uint32_t* sg = reinterpret_cast<uint32_t*>(p.scratch + (size_t)slot * G * p.kc * 12 + (size_t)G * p.kc * 8) +
                       (size_t)g * p.kc;
        const uint32_t kt = s_kt[g];
        const float* fcs = a.fcent + (size_t)slot * a.cap_clusters * D;
        uint32_t* hw = hist1 + g * 256;  // 16-bit keys are dead: histograms in the head's own area
        __shared__ uint32_t s_hc[GQ][256];
        uint32_t* hc = s_hc[g];
        unsigned long long rmn = ~0ull, rmx = 0ull;
        for (uint32_t i = gt; i < nc; i += GT) {
            const bool in = keys[g * p.kc + i] <= kt;
            unsigned long long kx = ~0ull;
            uint32_t w = 0;
            if (in) {
                uint32_t k, l;
                cand_of(i, k, l);
                const uint32_t cid = s_uu[k][2] + l;
                const float4* cv = reinterpret_cast<const float4*>(fcs + (size_t)cid * D);
                double sacc = 0.0;
                for (uint32_t j0 = 0; j0 < D / 4; j0 += 8) {
                    float4 v4[8];
#pragma unroll
                    for (uint32_t t = 0; t < 8; ++t) v4[t] = __ldg(cv + j0 + t);
#pragma unroll
                    for (uint32_t t = 0; t < 8; ++t) {
                        const uint32_t jq = j0 + t;
                        sacc = __fma_rn(s_qd[g * D + 4 * jq + 0], (double)v4[t].x, sacc);
                        sacc = __fma_rn(s_qd[g * D + 4 * jq + 1], (double)v4[t].y, sacc);
                        sacc = __fma_rn(s_qd[g * D + 4 * jq + 2], (double)v4[t].z, sacc);
                        sacc = __fma_rn(s_qd[g * D + 4 * jq + 3], (double)v4[t].w, sacc);
                    }
                }
                kx = desc_key(__dadd_rn(sacc, __dmul_rn(s_qn[g], a.frad[(size_t)slot * a.cap_clusters + cid])));
                w = p.mode == 1 ? ftok_g[cid] : 1u;
                rmn = min(rmn, kx);
                rmx = max(rmx, kx);
            }
            kg[i] = kx;
            sg[i] = w;
        }
        __shared__ unsigned long long s_rmn[GQ], s_rmx[GQ], s_prefix[GQ], s_mask[GQ];
        __shared__ uint32_t s_state[GQ], s_cbefore[GQ];
        __shared__ int s_shift[GQ];
        if (gt == 0) {
            s_rmn[g] = ~0ull;
            s_rmx[g] = 0ull;
        }
        bar_named(hbar, GT);
        atomicMin(&s_rmn[g], rmn);
        atomicMax(&s_rmx[g], rmx);
        bar_named(hbar, GT);
        if (gt == 0) {
            const unsigned long long mn = s_rmn[g], mx = s_rmx[g];
            const unsigned long long diff = mn ^ mx;
            const int top = diff ? 63 - __clzll((long long)diff) : 0;
            const int shift = top >= 7 ? top - 7 : 0;
            const unsigned long long mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
            s_prefix[g] = mn & mask;
            s_mask[g] = mask;
            s_shift[g] = shift;
            s_wbefore[g] = 0;
            s_state[g] = 0;
            s_nsel[g] = 0;
            s_cbefore[g] = 0;
        }
        for (;;) {
            bar_named(hbar, GT);
            const int shift = s_shift[g];
            if (s_state[g] != 0 || shift < 0) break;
            for (uint32_t b = gt; b < 256; b += GT) hw[b] = hc[b] = 0;
            bar_named(hbar, GT);
            const unsigned long long prefix = s_prefix[g], mask = s_mask[g];
            for (uint32_t i = gt; i < nc; i += GT) {
                const unsigned long long kv = kg[i];
                if (kv != ~0ull && (kv & mask) == prefix) {
                    atomicAdd(&hw[(uint32_t)(kv >> shift) & 255u], sg[i]);
                    atomicAdd(&hc[(uint32_t)(kv >> shift) & 255u], 1u);
                }
            }
            bar_named(hbar, GT);
            if (gt < 32) {
                uint32_t w8[8], c8[8];
                unsigned long long lw = 0;
                uint32_t lc = 0;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    w8[t] = hw[gt * 8 + t];
                    c8[t] = hc[gt * 8 + t];
                    lw += w8[t];
                    lc += c8[t];
                }
                unsigned long long iw = lw;
                uint32_t ic = lc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long yw = __shfl_up_sync(0xffffffffu, iw, o);
                    const uint32_t yc = __shfl_up_sync(0xffffffffu, ic, o);
                    if (gt >= (uint32_t)o) {
                        iw += yw;
                        ic += yc;
                    }
                }
                int found = -1;
                unsigned long long cum = s_wbefore[g] + (iw - lw), wexcl = 0;
                uint32_t ccum = ic - lc, cexcl = 0;
#pragma unroll
                for (int t = 0; t < 8; ++t)
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
                const unsigned int ballot = __ballot_sync(0xffffffffu, found >= 0);
                if (ballot == 0) {
                    if (gt == 0) s_state[g] = 2;
                } else if ((int)gt == __ffs(ballot) - 1) {
                    const uint32_t b = gt * 8 + (uint32_t)found;
                    s_prefix[g] = prefix | ((unsigned long long)b << shift);
                    s_mask[g] = mask | (255ull << shift);
                    s_wbefore[g] = wexcl;
                    s_cbefore[g] += cexcl;
                    s_state[g] = c8[found] == 1 ? 1u : 0u;
                    s_shift[g] = shift >= 8 ? shift - 8 : (shift > 0 ? 0 : -1);
                }
            }
        }
        bar_named(hbar, GT);
        const unsigned long long prefix = s_prefix[g], mask = s_mask[g];
        const uint32_t state = s_state[g], cbefore = s_cbefore[g];
        // the admitted candidates: below the boundary key, plus the boundary bucket when
        // it is the lone first element or everything fits
        for (uint32_t base = 0; base < nc; base += GT) {
            const uint32_t i = base + gt;
            bool take = false;
            if (i < nc && kg[i] != ~0ull) {
                const unsigned long long k = kg[i] & mask;
                take = k < prefix || (k == prefix && (state == 2 || (state == 1 && cbefore == 0)));
            }
            const unsigned int bal = __ballot_sync(0xffffffffu, take);
            uint32_t pos = 0;
            if (lane == 0 && bal) pos = atomicAdd(&s_nsel[g], (uint32_t)__popc(bal));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            bar_named(hbar, GT);  // the list overwrites weights other threads may still read
            if (take) sg[pos + __popc(bal & ((1u << lane) - 1u))] = i;
            bar_named(hbar, GT);
        }
        auto cid_of = [&](uint32_t i) -> uint32_t {
            uint32_t k, l;
            cand_of(i, k, l);
            return s_uu[k][2] + l;
        };
        if (state == 0 && gt == 0) {  // identical fp64 scores: reference-id order (retriever.cpp:33)
            unsigned long long used = s_wbefore[g];
            uint32_t admitted = cbefore, last_id = 0;
            bool first = true;
            for (;;) {
                int best = -1;
                uint32_t best_id = 0xffffffffu;
                for (uint32_t i = 0; i < nc; ++i) {
                    if (kg[i] == ~0ull || (kg[i] & mask) != prefix) continue;
                    const uint32_t oid = fo[cid_of(i)];
                    if ((first || oid > last_id) && oid < best_id) {
                        best_id = oid;
                        best = (int)i;
                    }
                }
                if (best < 0) break;
                const unsigned long long w = p.mode == 1 ? ftok_g[cid_of((uint32_t)best)] : 1ull;
                if (admitted > 0 && used + w > budget) break;
                used += w;
                ++admitted;
                sg[s_nsel[g]++] = (uint32_t)best;
                last_id = best_id;
                first = false;
            }
        }
        bar_named(hbar, GT);
        const uint32_t nsel = s_nsel[g];
        for (uint32_t x2 = gt; x2 < nsel; x2 += GT) {
            const uint32_t i = sg[x2], ci = cid_of(i);
            const unsigned long long ki = kg[i];
            const uint32_t oi = fo[ci];
            uint32_t rank = 0;
            for (uint32_t y = 0; y < nsel; ++y) {
                const unsigned long long ky = kg[sg[y]];
                if (ky < ki) ++rank;
                else if (ky == ki && y != x2 && fo[cid_of(sg[y])] < oi) ++rank;
            }
            out_cl[rank] = oi;
            if (grafted) atomicOr(&clb[ci >> 5], 1u << (ci & 31));
            for (uint32_t t = moff_g[ci]; t < moff_g[ci + 1]; ++t) {
                const uint32_t j = mem[t];
                atomicOr(&cb[j >> 5], 1u << (j & 31));
            }
        }
    }
    if (in_head) {
        bar_named(hbar, GT);
        // grafted chunks [m0, M) are not in the member CSR: test their clusters
        if (grafted) {
            __threadfence_block();
            const uint32_t* cc = a.chunk_clu + (size_t)slot * a.cap_chunks;
            for (uint32_t j = st.m0 + gt; j < M; j += GT) {
                const uint32_t cl = cc[j];
                if ((__ldcg(&clb[cl >> 5]) >> (cl & 31)) & 1u) atomicOr(&cb[j >> 5], 1u << (j & 31));
            }
        }
        if (gt == 0) {
            qi[g].n_units = kU;
            qi[g].n_clusters = s_nsel[g];
            qi[g].degenerate = 0;
            qi[g].error = 0;
            qi[g].scanned = (unsigned long long)P + nc;
        }
    }
    __syncthreads();
    FU_MARK(4)
    // ------------------------------------------------------------------ P4
    {
        const uint32_t ce = st.chunked_end, all = (1u << G) - 1u;
        Span* sp = a.spans + (size_t)slot * a.cap_spans;
        uint32_t* so = a.span_off + (size_t)slot * (a.cap_spans + 1);
        unsigned long long* sb = a.step_bytes + (size_t)slot * 4;
        uint32_t* rows = a.rows + (size_t)slot * a.cap_tokens;
        const unsigned long long dd = D;
        __shared__ uint32_t s_cnt[GQ], s_nsp[GQ];
        uint32_t* s_bnd = reinterpret_cast<uint32_t*>(sm);                   // [33][kFuThreads]
        uint32_t* s_sst = s_bnd + 33 * kFuThreads;                           // [kFuSpCache]
        uint32_t* s_slm = s_sst + kFuSpCache;
        uint32_t* s_soff = s_slm + kFuSpCache;
        if (tid < G) {
            s_cnt[tid] = 0;
            s_nsp[tid] = 0;
        }
        __syncthreads();
        const uint32_t mw = bit_words(M);
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
            for (uint32_t t = tid; t < sink_end; t += kFuThreads) rows[t] = t | (all << 24);
        }
        const uint32_t* cs = a.chunk_start + (size_t)slot * (a.cap_chunks + 1);
        uint32_t my_cnt[GQ], my_nsp[GQ];
#pragma unroll
        for (int h = 0; h < GQ; ++h) my_cnt[h] = my_nsp[h] = 0;
        for (uint32_t w0 = 0; w0 < mw; w0 += kFuThreads) {
            const uint32_t w = w0 + tid;
            uint32_t wg[GQ], any = 0;
#pragma unroll
            for (int h = 0; h < GQ; ++h) {
                wg[h] = w < mw ? cbits[h * mwcap + w] : 0u;
                any |= wg[h];
            }
            {
                uint32_t bnd[33];
#pragma unroll
                for (int b = 0; b <= 32; ++b) {
                    const bool need = (b < 32 && ((any >> b) & 1u)) || (b > 0 && ((any >> (b - 1)) & 1u));
                    bnd[b] = need ? __ldg(cs + w * 32 + b) : 0u;
                }
#pragma unroll
                for (int b = 0; b <= 32; ++b) s_bnd[b * kFuThreads + tid] = bnd[b];
            }
            uint32_t cnt = 0, toks = 0;
            for (uint32_t bits = any; bits; bits &= bits - 1u) {
                const uint32_t b = __ffs(bits) - 1;
                const uint32_t s0 = max(s_bnd[b * kFuThreads + tid], sink_end), e0 = s_bnd[(b + 1) * kFuThreads + tid];
                if (s0 < e0) {
                    ++cnt;
                    toks += e0 - s0;
                }
            }
            unsigned long long total;
            const unsigned long long ex = fu_scan<unsigned long long>(((unsigned long long)cnt << 40) | toks, s_wtot, total);
            uint32_t pos = out + (uint32_t)(ex >> 40), tp = tok + (uint32_t)(ex & 0xffffffffffull);
            for (uint32_t bits = any; bits; bits &= bits - 1u) {
                const uint32_t b = __ffs(bits) - 1;
                const uint32_t s0 = max(s_bnd[b * kFuThreads + tid], sink_end), e0 = s_bnd[(b + 1) * kFuThreads + tid];
                if (s0 >= e0) continue;
                uint32_t m = 0;
#pragma unroll
                for (int h = 0; h < GQ; ++h)
                    if ((wg[h] >> b) & 1u) {
                        m |= 1u << h;
                        my_cnt[h] += e0 - s0;
                        my_nsp[h] += 1;
                    }
                if (pos < a.cap_spans) {
                    sp[pos].start = s0;
                    sp[pos].len_mask = ((e0 - s0) << 8) | m;
                    so[pos] = tp;
                }
                if (pos < kFuSpCache) {
                    s_sst[pos] = s0;
                    s_slm[pos] = ((e0 - s0) << 8) | m;
                    s_soff[pos] = tp;
                }
                ++pos;
                tp += e0 - s0;
            }
            out += (uint32_t)(total >> 40);
            tok += (uint32_t)(total & 0xffffffffffull);
        }
#pragma unroll
        for (int h = 0; h < GQ; ++h) {
            const uint32_t c1 = __reduce_add_sync(0xffffffffu, my_cnt[h]);
            const uint32_t c2 = __reduce_add_sync(0xffffffffu, my_nsp[h]);
            if (lane == 0) {
                atomicAdd(&s_cnt[h], c1);
                atomicAdd(&s_nsp[h], c2);
            }
        }
        const uint32_t n_chunk_spans = out - (sink_end > 0 ? 1u : 0u);
        __syncthreads();
        {  // row list of the chunk spans: one thread per span writes its rows
            const uint32_t first = sink_end > 0 ? 1u : 0u, lim = min(out, a.cap_spans);
            for (uint32_t k = first + tid; k < lim; k += kFuThreads) {
                uint32_t s0, lm, off;
                if (k < kFuSpCache) {
                    s0 = s_sst[k];
                    lm = s_slm[k];
                    off = s_soff[k];
                } else {
                    s0 = sp[k].start;
                    lm = sp[k].len_mask;
                    off = so[k];
                }
                const uint32_t len = lm >> 8, hm = (lm & 0xffu) << 24;
                for (uint32_t t = 0; t < len; ++t) rows[off + t] = (s0 + t) | hm;
            }
        }
        if (p.flags == 1u) {  // buffer_ids = [chunked_end, n), disjoint from the chunks
            const uint32_t b0 = max(ce, sink_end);
            if (n > b0) {
                if (tid == 0 && out < a.cap_spans) {
                    sp[out].start = b0;
                    sp[out].len_mask = ((n - b0) << 8) | all;
                    so[out] = tok;
                }
                for (uint32_t t = tid; t < n - b0; t += kFuThreads) rows[tok + t] = (b0 + t) | (all << 24);
                ++out;
                tok += n - b0;
            }
        } else if (p.flags == 2u) {  // explicit sorted unique ids
            const uint32_t lo = p.buf_off[slot], hi = p.buf_off[slot + 1];
            for (uint32_t base = lo; base < hi; base += kFuThreads) {
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
                            uint32_t m = 0;
#pragma unroll
                            for (int hh = 0; hh < GQ; ++hh) m |= ((cbits[hh * mwcap + (l >> 5)] >> (l & 31)) & 1u) << hh;
                            resid = all & ~m;
                        }
                    }
                }
                unsigned long long total;
                const unsigned long long ex = fu_scan<unsigned long long>(resid ? ((1ull << 40) | 1ull) : 0ull, s_wtot, total);
                if (resid) {
                    rows[tok + (uint32_t)(ex & 0xffffffffffull)] = id | (resid << 24);
                    const uint32_t pos = out + (uint32_t)(ex >> 40);
                    if (pos < a.cap_spans) {
                        sp[pos].start = id;
                        sp[pos].len_mask = (1u << 8) | resid;
                        so[pos] = tok + (uint32_t)(ex & 0xffffffffffull);
                    }
#pragma unroll
                    for (int hh = 0; hh < GQ; ++hh)
                        if ((resid >> hh) & 1u) atomicAdd(&s_cnt[hh], 1u);
                }
                out += (uint32_t)(total >> 40);
                tok += (uint32_t)(total & 0xffffffffffull);
            }
        }
        if (p.aq.ctl) __threadfence();  // every thread's row-list writes, before the publication
        __syncthreads();
        if (tid == 0) {
            if (out > a.cap_spans) {
                atomicOr(a.err, kErrSpanOverflow);
                out = a.cap_spans;
            }
            so[out] = tok;
            a.n_spans[slot] = out;
            a.slot_tok[slot] = tok;
            const unsigned long long Pl = P;
            const uint32_t bufl = (p.flags == 1u && n > max(ce, sink_end)) ? n - max(ce, sink_end) : 0u;
            unsigned long long per_q = 0;
            for (uint32_t h = 0; h < G; ++h) {
                const unsigned long long act = (unsigned long long)s_cnt[h] + sink_end + bufl;
                qi[h].n_active = act;
                per_q += Pl * (4 * dd + 8) + (unsigned long long)s_nc[h] * (4 * dd + 16) +
                         (unsigned long long)s_nsp[h] * 8 + act * 2 * dd * 2 + 8 * dd;
            }
            const unsigned long long ncu = s_ncu;
            sb[0] = Pl * (4 * dd + 8) + ncu * (4 * dd + 16) + (unsigned long long)n_chunk_spans * 8 +
                    (unsigned long long)tok * 2 * dd * 2 + G * 8 * dd;
            sb[1] = per_q;
            sb[2] = tok;
            sb[3] = ncu;
        }
        if (p.aq.ctl && warp == 0) publish_tasks(p.aq, blockIdx.x, tok, aq_epoch, a.err);
    }
    FU_MARK(5)
    if (p.prof && tid == 0) p.prof[(size_t)slot * 16 + 6] = nstage | ((unsigned long long)s_rbase[G] << 32);
}

// ---------------------------------------------------------------------------
// Host: shape check, shared-memory sizing, launch.  Returns cudaErrorNotSupported
// when the shape does not fit (the caller then runs the four-kernel chain).
static uint32_t fu_region_a(uint32_t G, uint32_t cap_units, uint32_t pmax) {
    const uint32_t p1 = kFuD * cap_units * 4 + cap_units * 8 + G * pmax * 8 + (pmax + 1) * 4 + pmax * 4 + 64;
    const uint32_t ring = kFuStages * kFuStageBytes;
    const uint32_t p3 = G * kFuLC * kFuRBytes + 16 * kFuColBytes;
    const uint32_t p4 = 33 * kFuThreads * 4 + 3 * kFuSpCache * 4;
    return (std::max(std::max(p1, ring), std::max(p3, p4)) + 127) & ~127u;
}

template <int GQ>
static cudaError_t launch_fused_g(const FusedParams& p, uint32_t n_slots, size_t smem, cudaStream_t stream) {
    static KernelCfg cfg;
    cudaError_t e = ensure_smem(k_select<GQ>, cfg, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(k_select<GQ>, dim3(n_slots), dim3(kFuThreads), smem, stream, p);
}

cudaError_t launch_fused(const Arena& a, const float* q, const float* q_in, uint32_t unit_topk, uint32_t mode,
                         uint32_t cluster_topk, unsigned long long budget, uint32_t sink, uint32_t flags,
                         const uint32_t* buf_off, const uint32_t* buf_ids, unsigned char* scratch, uint32_t kc,
                         uint32_t uc, uint32_t pmax, uint32_t max_fanout, uint32_t n_slots, cudaStream_t stream,
                         const AttQueueDev* aq) {
    if (a.d != (uint32_t)kFuD || getenv("LC_NO_FUSED")) return cudaErrorNotSupported;
    if (max_fanout >= 16384) return cudaErrorNotSupported;  // stage descriptors hold 14-bit unit offsets
    if (a.G != 1 && a.G != 2 && a.G != 4 && a.G != 8) return cudaErrorNotSupported;
    if (unit_topk > kFuMaxKU || kc > 16384 || uc > 65535 || a.cap_tokens >= (1u << 24)) return cudaErrorNotSupported;
    if (std::min<uint64_t>((uint64_t)a.G * std::min(unit_topk, pmax), pmax) > kFuMaxUnion) return cudaErrorNotSupported;
    kc = (kc + 7) & ~7u;
    uc = (uc + 7) & ~7u;
    const uint32_t smem_a = fu_region_a(a.G, a.cap_units, pmax);
    const FuLayout lay = fu_layout(smem_a, a.G, kc, uc, bit_words(a.cap_chunks));
    const DevProps dp = dev_props();
    // static shared memory of the instantiation is below 24 KB; keep the total within the opt-in limit
    if ((size_t)lay.total + 24 * 1024 > (size_t)dp.smem_blk) return cudaErrorNotSupported;
    if (getenv("LC_FUSED_DEBUG")) {
        static int once = 0;
        if (!once++) {
            int occ = 0;
            if (a.G == 4) {
                static KernelCfg c4;
                ensure_smem(k_select<4>, c4, lay.total);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select<4>, kFuThreads, lay.total);
            }
            fprintf(stderr, "[k_select] kc %u uc %u pmax %u region A %u dynamic smem %u CTAs/SM %d\n", kc, uc, pmax,
                    smem_a, lay.total, occ);
        }
    }
    static unsigned long long* prof_dev[kMaxDevices] = {};
    const bool want_prof = getenv("LC_PROF") != nullptr;
    unsigned long long*& prof = prof_dev[current_device()];
    if (want_prof && !prof) {
        cudaMalloc(&prof, (size_t)a.n_slots * 16 * 8);
        cudaMemset(prof, 0, (size_t)a.n_slots * 16 * 8);
    }
    FusedParams fp{a, q, q_in ? q_in : q, unit_topk, mode, cluster_topk, sink, flags, budget, buf_off, buf_ids,
                   scratch, kc, uc, smem_a, fu_g8cap(uc), 0u, want_prof ? prof : nullptr,
                   aq ? *aq : AttQueueDev{}};
    if (const char* ev = getenv("LC_FUSED_PF")) fp.pf = (uint32_t)atoi(ev);  // experiments
    cudaError_t e;
    switch (a.G) {
        case 1: e = launch_fused_g<1>(fp, n_slots, lay.total, stream); break;
        case 2: e = launch_fused_g<2>(fp, n_slots, lay.total, stream); break;
        case 4: e = launch_fused_g<4>(fp, n_slots, lay.total, stream); break;
        default: e = launch_fused_g<8>(fp, n_slots, lay.total, stream); break;
    }
    if (want_prof && e == cudaSuccess) {  // diagnostics: per-phase means and the slowest slot
        cudaStreamSynchronize(stream);
        std::vector<unsigned long long> t((size_t)a.n_slots * 16);
        cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
        double ph[5] = {0, 0, 0, 0, 0}, mx = 0, cnt = 0, st = 0, rr = 0;
        unsigned long long t0 = ~0ull, t1 = 0;
        for (uint32_t s = a.slot0; s < a.slot0 + n_slots; ++s) {
            const unsigned long long* x = &t[(size_t)s * 16];
            if (!x[5] || x[5] < x[0]) continue;
            for (int k = 0; k < 5; ++k) ph[k] += (double)(x[k + 1] - x[k]);
            mx = std::max(mx, (double)(x[5] - x[0]));
            t0 = std::min(t0, x[0]);
            t1 = std::max(t1, x[5]);
            st += (double)(x[6] & 0xffffffffull);
            rr += (double)(x[6] >> 32);
            cnt += 1;
        }
        double sub[7] = {0, 0, 0, 0, 0, 0, 0};
        for (uint32_t s = a.slot0; s < a.slot0 + n_slots; ++s) {
            const unsigned long long* x = &t[(size_t)s * 16];
            if (!x[5] || x[5] < x[0]) continue;
            sub[0] += (double)(x[8] - x[0]);   // q + coarse staging
            sub[1] += (double)(x[9] - x[8]);   // chains + norms
            sub[2] += (double)(x[10] - x[9]);  // keys + rank
            sub[3] += (double)(x[1] - x[10]);  // union + group table
            sub[4] += (double)(x[11] - x[2]);  // digits, list, R
            sub[5] += (double)(x[12] - x[11]); // R concatenation
            sub[6] += (double)(x[3] - x[12]);  // exact chains
        }
        if (cnt > 0)
            fprintf(stderr, "[LC_PROF] k_select detail us: stage %.2f chains %.2f rank %.2f union %.2f | list+R %.2f "
                    "concat %.2f exact %.2f\n", sub[0] / cnt / 1e3, sub[1] / cnt / 1e3, sub[2] / cnt / 1e3,
                    sub[3] / cnt / 1e3, sub[4] / cnt / 1e3, sub[5] / cnt / 1e3, sub[6] / cnt / 1e3);
        if (cnt > 0)
            fprintf(stderr, "[LC_PROF] k_select per-CTA us: coarse %.2f fine %.2f select(x,R) %.2f rank+members %.2f "
                    "spans %.2f | max %.2f | first start->last end %.1f us | stages %.1f R %.1f per slot\n",
                    ph[0] / cnt / 1e3, ph[1] / cnt / 1e3, ph[2] / cnt / 1e3, ph[3] / cnt / 1e3, ph[4] / cnt / 1e3,
                    mx / 1e3, (double)(t1 - t0) / 1e3, st / cnt, rr / cnt);
        if (cnt > 0) {  // the slowest decile of CTAs: where their time goes and how big their slots are
            std::vector<std::pair<double, uint32_t>> dur;
            for (uint32_t s = a.slot0; s < a.slot0 + n_slots; ++s) {
                const unsigned long long* x = &t[(size_t)s * 16];
                if (x[5] && x[5] >= x[0]) dur.push_back({(double)(x[5] - x[0]), s});
            }
            std::sort(dur.begin(), dur.end());
            const size_t k0 = dur.size() - std::max<size_t>(1, dur.size() / 10);
            double sp[5] = {0, 0, 0, 0, 0}, sst = 0, srr = 0, c2 = 0, start = 0;
            for (size_t i = k0; i < dur.size(); ++i) {
                const unsigned long long* x = &t[(size_t)dur[i].second * 16];
                for (int k = 0; k < 5; ++k) sp[k] += (double)(x[k + 1] - x[k]);
                sst += (double)(x[6] & 0xffffffffull);
                srr += (double)(x[6] >> 32);
                start += (double)(x[0] - t0);
                c2 += 1;
            }
            fprintf(stderr, "[LC_PROF] k_select slowest 10%%: coarse %.2f fine %.2f select %.2f rank+members %.2f spans "
                    "%.2f us | start offset %.2f us | stages %.1f R %.1f | median CTA %.2f us\n",
                    sp[0] / c2 / 1e3, sp[1] / c2 / 1e3, sp[2] / c2 / 1e3, sp[3] / c2 / 1e3, sp[4] / c2 / 1e3,
                    start / c2 / 1e3, sst / c2, srr / c2, dur[dur.size() / 2].first / 1e3);
        }
    }
    return e;
}

}  // namespace lc
