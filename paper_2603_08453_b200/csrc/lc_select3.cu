// Three-kernel selection pipeline (north star item 2), one phase per kernel so
// that each phase runs with the parallelism it needs:
//
//   k_coarse  (one CTA per slot): ||q_g|| and the coarse tier for all G query
//             heads of the GQA group (retriever.cpp:97-116), per-head top-k_g
//             units, and the union of the kept units with each head's
//             candidate offsets -> a small per-slot plan in global memory.
//   k_fine    (one warp per 32 union candidates, grid over all slots): each lane
//             loads its candidate's whole centroid (one [d/4][n_u][4] column,
//             512-byte lines across the warp) into registers, then runs one
//             sequential fp64 chain per head that kept the unit -- bit-exact
//             kernels::dot, upper bound dot + ||q||*r (kernels.cpp:155-159).
//             Pure streaming: every centroid of the union is read once.
//   k_pick    (one CTA per slot): per head, on its own warps, the exact
//             weighted radix select of the token-budget prefix / fixed k_c
//             (retriever.cpp:140-154) and the rank sort of the selection; then
//             the union active spans from the member lists of the selected
//             clusters (collect_active, retriever.cpp:60-74).
#include "lc_common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lc {

namespace {

constexpr int kMaxKU3 = 64;

// plan layout (bytes): 0: u32 degenerate, nuu, ncu, kU, nc[8]; 64: u64 kmin[8];
// 128: u64 kmax[8]; 192: f64 qnorm[8]; 256: units u32 [cap_units][4 + G] =
// unit, mask, base, n_u, qoff[G]; then ucum u32 [cap_units + 1] (first union
// candidate of each union unit); then, 16-byte aligned, q as f64 [G][D]
// (plan_layout() is the single definition, shared with the host)
struct PlanView {
    unsigned char* b;
    uint32_t ucum_off, qd_off, tile_off;
    __device__ PlanView(unsigned char* base, const Arena& a) : b(base) {
        plan_layout(a.cap_units, a.G, a.d, a.cap_clusters, &ucum_off, &qd_off, &tile_off);
    }
    __device__ uint32_t* hdr() const { return reinterpret_cast<uint32_t*>(b); }
    __device__ unsigned long long* kmin() const { return reinterpret_cast<unsigned long long*>(b + 64); }
    __device__ unsigned long long* kmax() const { return reinterpret_cast<unsigned long long*>(b + 128); }
    __device__ double* qnorm() const { return reinterpret_cast<double*>(b + 192); }
    __device__ uint32_t* units() const { return reinterpret_cast<uint32_t*>(b + 256); }
    __device__ uint32_t* ucum() const { return reinterpret_cast<uint32_t*>(b + ucum_off); }
    __device__ double* qd() const { return reinterpret_cast<double*>(b + qd_off); }
    __device__ uint4* tiles() const { return reinterpret_cast<uint4*>(b + tile_off); }
};

// inverse of desc_key: the score a key stands for
__device__ __forceinline__ double key_score(unsigned long long key) {
    const unsigned long long ord = ~key;
    const unsigned long long b = (ord >> 63) ? (ord & 0x7fffffffffffffffull) : ~ord;
    return __longlong_as_double((long long)b);
}

constexpr uint32_t kPickRCap = 128;   // refinement list kept in shared memory
constexpr uint32_t kPickCols = 8;     // refinement centroids staged per pass
constexpr uint32_t kPickBufs = 2;     // ... double-buffered
constexpr uint32_t kPickStage = 256;  // rank-phase staging entries
// k_pickq's phase buffer: the radix histograms, the refinement (centroid
// columns + the per-R arrays) and the rank phase's staging live in different
// phases of the kernel and share one static buffer.
template <int DQ>
struct PickPhase {
    static constexpr uint32_t refine = kPickBufs * kPickCols * (DQ + 4) * 4 + kPickRCap * (8 + 8 + 6 * 4);
    static constexpr uint32_t stage = kPickStage * 16, hist = 2 * 256 * 4;
    static constexpr uint32_t bytes =
        refine > stage ? (refine > hist ? refine : hist) : (stage > hist ? stage : hist);
};

__device__ __forceinline__ void bar_g(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

}  // namespace

// 1D TMA (cp.async.bulk) into shared memory with mbarrier completion
__device__ __forceinline__ void bulk_g2s3(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init3(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect3(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait3(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void mma_f16x(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2x(float lo, float hi) {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
// the tensor-core filter's error constants (the same computation and bound as
// k_select, lc_fused.cu): fp16 rounding of c (2^-11), q's fp16 hi + lo split
// (2^-22), fp32 MMA accumulation over <= 16 k-steps (2^-15, generous), the
// final hi + lo add (2^-24), subnormal terms 2^-25 sqrt(d); 2^-44 for the
// reference's fp64 dot and our fp64 adds
constexpr double kFiK1 = 5.25e-4;
constexpr double kFiK2 = 3.5e-7;
constexpr double kFiK3 = 5.7e-14;

struct Sel3Params {
    Arena a;
    uint32_t keys_cap;  // per-head candidates staged in k_pickq's shared memory
    const float* q;  // [slot][G][d]
    const float* q_in;  // k_coarse's source of q when it differs (host-mapped); k_coarse copies it to q
    uint32_t unit_topk, mode, cluster_topk, sink, flags;
    unsigned long long budget;
    const uint32_t* buf_off;
    const uint32_t* buf_ids;
    unsigned char* scratch;  // per slot: keys u64 [G][qcap] + weights/selection u32 [G][qcap]
    uint32_t qcap;
    unsigned long long* prof;  // optional k_pick phase timestamps [slot][8] (LC_PROF=1)
    uint32_t* fine_ctr;        // k_fine pool / exit counters [0, 2) (reset by k_fine); k_pickq's
                               // size-class counters [16, 32) (reset by k_spans); zeroed
    uint32_t* pick_ord;        // k_pickq's heads by size class: [class][n_slots * G] (this group)
    unsigned long long* prof_sp;  // optional k_spans phase timestamps [slot][8] (LC_PROF=1)
};

__device__ __forceinline__ unsigned long long gtime3() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define LC_PMARK(ph) \
    if (p.prof && threadIdx.x == 0) p.prof[((size_t)slot * GQ + g) * 8 + (ph)] = gtime3();

// ---------------------------------------------------------------------------
constexpr int kCoThreads = 256;

// k_pickq's launch order: k_coarse files every (slot, head) under the log2 size
// class of its candidate count, and k_pickq's CTAs take the heads largest class
// first, so the few long heads start in the first wave instead of ending the
// kernel (longest-processing-time-first list scheduling).
constexpr uint32_t kPickClasses = 16;
__device__ __forceinline__ uint32_t pick_class(uint32_t nc) {
    const uint32_t c = nc ? 31u - __clz(nc) : 0u;
    return kPickClasses - 1u - min(c, kPickClasses - 1u);  // class 0: the largest heads
}
__device__ __forceinline__ void pick_push(const Sel3Params& p, uint32_t h, uint32_t nc) {
    const uint32_t c = pick_class(nc), nh = gridDim.x * p.a.G;  // k_coarse: one CTA per slot
    const uint32_t at = atomicAdd(p.fine_ctr + 16 + c, 1u);
    if (at < nh) p.pick_ord[(size_t)c * nh + at] = h;  // (a miscount falls back to launch order)
}

template <int D, int GQ>
__global__ void __launch_bounds__(kCoThreads) k_coarse(Sel3Params p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Arena& a = p.a;
    const uint32_t slot = a.slot0 + blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t G = GQ, d = D;
    const SlotState st = a.state[slot];
    const uint32_t n = st.n_tokens, P = st.P;
    PlanView pv(a.plan + (size_t)slot * a.plan_bytes, a);
    const bool degenerate = (p.mode == 1 && (unsigned long long)n <= p.budget) || st.n_chunks == 0;
    if (degenerate) {
        if (p.q_in != p.q)  // k_attend still reads this slot's q (full attention)
            for (uint32_t x = tid; x < G * D; x += kCoThreads)
                const_cast<float*>(p.q)[(size_t)slot * G * D + x] = p.q_in[(size_t)slot * G * D + x];
        if (tid == 0) {
            pv.hdr()[0] = 1;
            pv.hdr()[1] = pv.hdr()[2] = 0;
        }
        if (tid < G) pick_push(p, blockIdx.x * G + tid, 0u);
        return;
    }
    const uint32_t Pp = (P + 3) & ~3u;
    double* qd = reinterpret_cast<double*>(smem);            // [G][D]
    float* ucs = reinterpret_cast<float*>(qd + G * D);       // [D][Pp]
    unsigned long long* ukey = reinterpret_cast<unsigned long long*>(ucs + (size_t)D * Pp);  // [G][P]
    double* s_urad = reinterpret_cast<double*>(ukey + (size_t)G * P);                         // [P]
    uint32_t* s_uoff = reinterpret_cast<uint32_t*>(s_urad + P);                              // [P + 1]
    uint32_t* s_umask = s_uoff + P + 1;                                                      // [P]
    __shared__ double s_qn[GQ];
    __shared__ uint32_t s_kept[GQ][kMaxKU3];
    __shared__ uint32_t s_ucum[1025];
    __shared__ uint32_t s_nuu;

    // every global input of the kernel is requested up front
    const double* ur = a.urad + (size_t)slot * a.cap_units;
    const uint32_t* uoff = a.unit_off + (size_t)slot * (a.cap_units + 1);
    for (uint32_t u = tid; u <= P; u += kCoThreads) {
        s_uoff[u] = uoff[u];
        if (u < P) {
            s_urad[u] = ur[u];
            s_umask[u] = 0;
        }
    }
    for (uint32_t x = tid; x < G * D; x += kCoThreads) {
        qd[x] = (double)p.q_in[(size_t)slot * G * D + x];
        pv.qd()[x] = qd[x];  // k_fine reads q as f64 from the plan (L1-resident)
    }
    const float* uc = a.ucent + (size_t)slot * a.cap_units * d;
    {
        // element e = (row j, float4 column c) of the [D][Pp] tile, walked
        // without a division per element
        const uint32_t pq = Pp >> 2, n4 = D * pq, sj = kCoThreads / pq, sc = kCoThreads % pq;
        uint32_t j = tid / pq, c = tid % pq;
        constexpr int kB = 8;
        for (uint32_t e0 = 0; e0 < n4; e0 += kB * kCoThreads) {
            float4 v[kB];
            uint32_t jj[kB], cc[kB];
#pragma unroll
            for (int t = 0; t < kB; ++t) {
                jj[t] = j;
                cc[t] = c;
                if (e0 + t * kCoThreads + tid < n4)
                    v[t] = __ldg(reinterpret_cast<const float4*>(uc + (size_t)j * a.cap_units) + c);
                j += sj;
                c += sc;
                if (c >= pq) {
                    c -= pq;
                    ++j;
                }
            }
#pragma unroll
            for (int t = 0; t < kB; ++t)
                if (e0 + t * kCoThreads + tid < n4) reinterpret_cast<float4*>(ucs + (size_t)jj[t] * Pp)[cc[t]] = v[t];
        }
    }
    __syncthreads();
    // one thread per unit runs the G coarse dots as independent chains (one
    // fp32->fp64 conversion of the centroid element feeds all of them);
    // ||q_g|| (kernels.cpp:19-23) runs on the last warp when it holds no unit
    const bool qn_apart = P <= kCoThreads - 32;
    if (qn_apart && warp == kCoThreads / 32 - 1) {
        if (lane < G) {
            double n2 = 0.0;
#pragma unroll 8
            for (uint32_t j = 0; j < d; ++j) n2 = __fma_rn(qd[lane * D + j], qd[lane * D + j], n2);
            s_qn[lane] = __dsqrt_rn(n2);
        }
    } else {
        for (uint32_t u = tid; u < P; u += kCoThreads) {
            double s[GQ];
#pragma unroll
            for (int g = 0; g < GQ; ++g) s[g] = 0.0;
#pragma unroll 4
            for (uint32_t j = 0; j < d; ++j) {
                const double c = (double)ucs[j * Pp + u];
#pragma unroll
                for (int g = 0; g < GQ; ++g) s[g] = __fma_rn(qd[g * D + j], c, s[g]);
            }
#pragma unroll
            for (int g = 0; g < GQ; ++g) ukey[g * P + u] = __double_as_longlong(s[g]);  // raw dot for now
        }
    }
    if (!qn_apart) {
        __syncthreads();
        if (tid < G) {
            double n2 = 0.0;
            for (uint32_t j = 0; j < d; ++j) n2 = __fma_rn(qd[tid * D + j], qd[tid * D + j], n2);
            s_qn[tid] = __dsqrt_rn(n2);
        }
    }
    __syncthreads();
    for (uint32_t x = tid; x < G * P; x += kCoThreads) {
        const uint32_t g = x / P, u = x % P;
        ukey[x] = desc_key(__dadd_rn(__longlong_as_double(ukey[x]), __dmul_rn(s_qn[g], s_urad[u])));
    }
    __syncthreads();
    const uint32_t kU = min(min(p.unit_topk, P), (uint32_t)kMaxKU3);
    for (uint32_t x = tid; x < G * P; x += kCoThreads) {
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
    // selected_units (rank order) and the union of kept units in ascending unit order
    for (uint32_t x = tid; x < G * kU; x += kCoThreads)
        a.sel_units[((size_t)slot * G + x / kU) * a.cap_units + x % kU] = s_kept[x / kU][x % kU];
    if (warp == 0) {
        uint32_t* uu = pv.units();
        const uint32_t stride = 4 + G;
        uint32_t pos = 0, ncu = 0;
        uint32_t qacc[GQ];
#pragma unroll
        for (int g = 0; g < GQ; ++g) qacc[g] = 0;
        for (uint32_t u0 = 0; u0 < P; u0 += 32) {
            const uint32_t u = u0 + lane;
            uint32_t m = u < P ? s_umask[u] : 0u;
            const uint32_t nu = m ? s_uoff[u + 1] - s_uoff[u] : 0u;
            if (nu == 0) m = 0;  // an empty unit contributes no candidate
            const unsigned int bal = __ballot_sync(0xffffffffu, m != 0);
            const uint32_t idx = pos + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
            for (int g = 0; g < GQ; ++g) {
                const uint32_t mine = ((m >> g) & 1u) ? nu : 0u;
                uint32_t x = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                if (m) uu[idx * stride + 4 + g] = qacc[g] + x - mine;
                qacc[g] += __shfl_sync(0xffffffffu, x, 31);
            }
            {
                uint32_t x = nu;  // nu == 0 for units outside the union
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                if (m) {
                    pv.ucum()[idx] = ncu + x - nu;
                    s_ucum[idx] = ncu + x - nu;
                }
            }
            if (m) {
                uu[idx * stride + 0] = u;
                uu[idx * stride + 1] = m;
                uu[idx * stride + 2] = s_uoff[u];
                uu[idx * stride + 3] = nu;
            }
            ncu += __reduce_add_sync(0xffffffffu, nu);
            pos += __popc(bal);
        }
        if (lane == 0) {
            pv.hdr()[0] = 0;
            pv.hdr()[1] = pos;
            pv.hdr()[2] = ncu;
            pv.hdr()[3] = kU;
            pv.ucum()[pos] = ncu;
            s_ucum[pos] = ncu;
            s_nuu = pos;
        }
        if (lane < G) {
            pv.hdr()[4 + lane] = qacc[lane];
            pick_push(p, blockIdx.x * G + lane, qacc[lane]);
            pv.kmin()[lane] = ~0ull;
            pv.kmax()[lane] = 0ull;
            pv.qnorm()[lane] = s_qn[lane];
        }
    }
    __syncthreads();
    // fine tile table: tile t covers union candidates [32t, 32t + 32)
    {
        const uint32_t nuu = s_nuu, ncu = s_ucum[nuu], ntiles = (ncu + 31) / 32;
        for (uint32_t t = tid; t < ntiles; t += kCoThreads) {
            const uint32_t c0 = t * 32;
            uint32_t lo = 0, hi = nuu;  // last unit with ucum <= c0
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_ucum[mid] <= c0) lo = mid;
                else hi = mid;
            }
            uint32_t mask = 0;
            for (uint32_t k = lo + 1; k < nuu && s_ucum[k] < c0 + 32; ++k) mask |= 1u << (s_ucum[k] - c0);
            pv.tiles()[t] = make_uint4(lo, mask, c0 - s_ucum[lo], min(32u, ncu - c0));
        }
    }
    // q read from a host-mapped buffer: leave the device copy the later kernels
    // read (stored last, so no load above waits behind a possibly aliasing store)
    if (p.q_in != p.q)
        for (uint32_t x = tid; x < G * D; x += kCoThreads) const_cast<float*>(p.q)[(size_t)slot * G * D + x] = (float)qd[x];
}

// ---------------------------------------------------------------------------
// k_fine: persistent fine-tier scoring, as a certified fp32 filter.
//
// The union candidates of every slot form one global list of 32-candidate
// tiles (slot-major; k_coarse planned each slot's union and its tile table).
// Each warp scores a contiguous static range of tiles, then claims single
// tiles from a pool (the last kFinePoolPct % of the list) as it finishes, so
// SMs that see less bandwidth do less work.  In a tile each lane owns one
// candidate.  A tile's fp16 rows are contiguous within each coarse unit, so
// the lane that starts a unit's run moves the whole run with one 1D TMA bulk
// copy into the warp's 3-stage shared-memory ring (mbarrier completion); two
// tiles are in flight while the warp scores the third, and no row sits in
// registers.
//
// The reference upper bound UB = fl64(sequential fp64 q.c) + qn*r
// (kernels.cpp:155-159) is enclosed, not computed, from the fp16 copy of the
// centroids (half the bytes): with c~ = fp16(c), s = fp32 q.c~ gives
// |UB_ref - UB~| <= e with UB~ = s + qn*r and
// e = ||q|| (1.01 * 132 * 2^-24 ||c|| + 2^-11 ||c|| + 2^-25 sqrt(d)) + 2^-49 |UB~|
// (fp16 rounding of c, recursive-summation bound for 128 products + 3
// partial-sum adds in fp32, the fp64 dot's and adds' roundings; ||c|| bounded
// from one fp32 sum of squares of c~ shared by every head).  k_pickq selects on the lower bounds, then recomputes the exact
// fp64 chain (bit-exact kernels::dot) only for candidates whose upper bound
// reaches the selection cut, so every selection stays bit-exact while the
// bulk of the scoring runs at fp32 speed.
constexpr int kFiThreads = 128;
constexpr int kFiWarps = kFiThreads / 32;
constexpr uint32_t kFinePoolPct = 10;
constexpr uint32_t kScratchEntry = 20;  // bytes per (head, candidate): lo key u64, weight u32, hi f64

template <int D, int GQ>
__global__ void __launch_bounds__(kFiThreads, 2) k_fine(Sel3Params p, uint32_t n) {
    pdl_wait();
    const Arena& a = p.a;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t G = GQ, V = D / 4;  // float4s per centroid
    __shared__ uint32_t s_tp[kMaxAttendSlots + 1];  // prefix of the slots' tile counts
    __shared__ uint32_t s_ws[kFiWarps];
    __shared__ __align__(8) unsigned long long s_fbar[kFiWarps][3];  // the warps' ring barriers
    __shared__ float s_sco[kFiWarps][GQ][32];                       // a tile's scores, (head, candidate)
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < 3; ++st) mbar_init3((uint32_t)__cvta_generic_to_shared(&s_fbar[warp][st]), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    {
        const uint32_t per = (n + kFiThreads - 1) / kFiThreads, i0 = tid * per;
        uint32_t loc = 0;
        for (uint32_t i = i0; i < i0 + per && i < n; ++i) {
            const uint32_t* h = reinterpret_cast<const uint32_t*>(a.plan + (size_t)(a.slot0 + i) * a.plan_bytes);
            loc += h[0] ? 0u : (h[2] + 31) / 32;
        }
        uint32_t x = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) s_ws[warp] = x;
        __syncthreads();
        uint32_t run = x - loc;
        for (uint32_t w = 0; w < warp; ++w) run += s_ws[w];
        if (tid == 0) s_tp[0] = 0;
        for (uint32_t i = i0; i < i0 + per && i < n; ++i) {
            const uint32_t* h = reinterpret_cast<const uint32_t*>(a.plan + (size_t)(a.slot0 + i) * a.plan_bytes);
            run += h[0] ? 0u : (h[2] + 31) / 32;
            s_tp[i + 1] = run;
        }
        __syncthreads();
    }
    const uint32_t TT = s_tp[n];
    uint32_t* ctr = p.fine_ctr;  // [0] next pool tile, [1] CTAs out
    if (TT > 0) {
        const uint32_t NW = gridDim.x * kFiWarps, w = blockIdx.x * kFiWarps + warp;
        const uint32_t TS = TT - (uint32_t)(((unsigned long long)TT * kFinePoolPct) / 100);
        uint32_t cur_t = (uint32_t)(((unsigned long long)TS * w) / NW);
        const uint32_t s_end = (uint32_t)(((unsigned long long)TS * (w + 1)) / NW);
        uint32_t claim = 0;  // lane 0: pool tile claimed one tile before it is needed
        if (cur_t >= s_end && lane == 0) claim = TS + atomicAdd(ctr, 1u);
        auto next_tile = [&]() -> uint32_t {
            if (cur_t < s_end) {
                const uint32_t t = cur_t++;
                if (cur_t >= s_end && lane == 0) claim = TS + atomicAdd(ctr, 1u);
                return t;
            }
            const uint32_t t = __shfl_sync(0xffffffffu, claim, 0);
            if (t >= TT) return ~0u;
            if (lane == 0) claim = TS + atomicAdd(ctr, 1u);
            return t;
        };
        uint32_t lo = 0;  // slot (local index) of the last looked-up tile
        // A tile goes through four steps, one loop iteration apart, so no
        // dependent load sits on the critical path: (A) slot lookup + tile-table
        // entry load, (B) the lane's unit row loads, (I) the bulk copy of the
        // tile's rows and their filter metadata (issued by the lanes that start
        // a unit run), (C) scoring from shared memory.
        struct StA {
            uint32_t slot, ti;  // slot ~0u: no tile
            uint4 te;           // {first unit, unit starts, first local, candidates in the tile}
        };
        struct StB {
            uint32_t slot, valid, local, base, mask, vc, starts;
            uint32_t qoff[GQ];
        };
        auto stage_a = [&](uint32_t t) -> StA {
            StA x;
            x.slot = ~0u;
            if (t == ~0u) return x;
            if (t < s_tp[lo] || t >= s_tp[lo + 1]) {
                uint32_t l = 0, h = n;
                while (h - l > 1) {
                    const uint32_t mid = (l + h) >> 1;
                    if (s_tp[mid] <= t) l = mid;
                    else h = mid;
                }
                while (s_tp[l + 1] <= t) ++l;
                lo = l;
            }
            x.slot = a.slot0 + lo;
            x.ti = t - s_tp[lo];
            const PlanView pv(a.plan + (size_t)x.slot * a.plan_bytes, a);
            x.te = __ldg(pv.tiles() + x.ti);
            return x;
        };
        auto stage_b = [&](const StA& x) -> StB {
            StB y;
            y.slot = x.slot;
            y.valid = 0;
            y.mask = 0;
            y.vc = 0;
            if (x.slot == ~0u) return y;
            const PlanView pv(a.plan + (size_t)x.slot * a.plan_bytes, a);
            y.vc = x.te.w;
            y.valid = lane < y.vc;
            y.starts = x.te.y;
            const uint32_t below = x.te.y & ((2u << lane) - 1u);  // unit starts at positions <= lane
            const uint32_t nb = __popc(below);
            const uint32_t k = x.te.x + nb;
            y.local = y.valid ? (nb ? lane - (31 - __clz(below)) : x.te.z + lane) : 0u;
            const uint32_t* u = pv.units() + (size_t)k * (4 + G);
            y.base = __ldg(u + 2);
            y.mask = y.valid ? __ldg(u + 1) : 0u;
#pragma unroll
            for (int g = 0; g < GQ; ++g) y.qoff[g] = __ldg(u + 4 + g);
            return y;
        };
        // the warp's ring: 3 stages of 32 rows + their 16-byte filter metadata
        // (radius, norm bound, token count); one barrier per stage
        constexpr uint32_t ROWB = D * 2, STG = 32 * ROWB, NSTG = 3, MSTG = 32 * 16;
        extern __shared__ __align__(128) unsigned char fsm[];
        const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(fsm + (size_t)warp * NSTG * STG);
        const uint32_t meta_s =
            (uint32_t)__cvta_generic_to_shared(fsm + (size_t)kFiWarps * NSTG * STG + (size_t)warp * NSTG * MSTG);
        const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&s_fbar[warp][0]);
        float* qs = reinterpret_cast<float*>(fsm + (size_t)kFiWarps * NSTG * (STG + MSTG)) + (size_t)warp * GQ * D;
        uint32_t qslot = ~0u, fslot = ~0u;
        constexpr int KSF = D >= 32 ? D / 16 : 2;  // MMA k-steps (D >= 32; smaller dims use fp32 FMAs)
        const uint32_t r = lane >> 2, c = lane & 3;
        uint32_t qf[KSF][4];
        // (I): the lanes that start a unit run copy the run's rows and metadata
        auto issue = [&](StB& y, uint32_t st) {
            if (y.slot == ~0u) return;
            const uint32_t bar = bar_s + 8u * st;
            if (lane == 0) mbar_expect3(bar, y.vc * (ROWB + 16u));
            __syncwarp();
            const bool start = y.valid && (lane == 0 || ((y.starts >> lane) & 1u));
            if (start) {
                const uint32_t later = y.starts & ~((2u << lane) - 1u);
                const uint32_t end = min(later ? (uint32_t)(__ffs(later) - 1) : 32u, y.vc);
                // the ring stage was read (generic proxy) before the warp's last __syncwarp
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                bulk_g2s3(ring_s + st * STG + lane * ROWB,
                          a.frow16 + (size_t)y.slot * a.cap_clusters * D + ((size_t)y.base + y.local) * D,
                          (end - lane) * ROWB, bar);
                bulk_g2s3(meta_s + st * MSTG + lane * 16u,
                          a.fmeta + (size_t)y.slot * a.cap_clusters + y.base + y.local, (end - lane) * 16u, bar);
            }
        };
        uint32_t mslot = ~0u;  // slot whose per-head key range the warp is tracking
        unsigned long long wmin[GQ], wmax[GQ];
        auto flush_minmax = [&]() {
            if (mslot == ~0u) return;
            PlanView pv(a.plan + (size_t)mslot * a.plan_bytes, a);
#pragma unroll
            for (int g = 0; g < GQ; ++g) {
                unsigned long long mn = wmin[g], mx = wmax[g];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                if (lane == 0 && mx != 0ull) {
                    atomicMin(pv.kmin() + g, mn);
                    atomicMax(pv.kmax() + g, mx);
                }
            }
        };

        // prologue: B of tiles 0..2, tiles 0 and 1 issued, A of tile 3
        StA sa = stage_a(next_tile());
        StB d = stage_b(sa);
        sa = stage_a(next_tile());
        StB n1 = stage_b(sa);
        issue(d, 0);
        sa = stage_a(next_tile());
        StB n2 = stage_b(sa);
        issue(n1, 1);
        sa = stage_a(next_tile());
        for (uint32_t it = 0; d.slot != ~0u; ++it) {
            issue(n2, (it + 2) % NSTG);       // (I) tile it + 2
            const StB nb = stage_b(sa);       // (B) tile it + 3
            sa = stage_a(next_tile());        // (A) tile it + 4
            if (D < 32 && d.slot != qslot) {  // the tile's q (fp32) into the warp's buffer
                __syncwarp();
                const float4* src = reinterpret_cast<const float4*>(p.q + (size_t)d.slot * G * D);
                for (uint32_t c = lane; c < G * D / 4; c += 32) reinterpret_cast<float4*>(qs)[c] = __ldg(src + c);
                qslot = d.slot;
                __syncwarp();
            }
            mbar_wait3(bar_s + 8u * (it % NSTG), (it / NSTG) & 1u);  // (C) this tile's rows
            if constexpr (D >= 32) {
            if (d.slot != fslot) {  // q as fp16 hi + lo rows of the MMA A operand (heads r, r + 8)
                fslot = d.slot;
                const uint32_t gr = r < G ? r : 0u;
#pragma unroll
                for (int s2 = 0; s2 < KSF; ++s2) {
                    const float4 q4 =
                        __ldg(reinterpret_cast<const float4*>(p.q + ((size_t)d.slot * G + gr) * D + c * (D / 4) + 4 * s2));
                    const float qq[4] = {q4.x, q4.y, q4.z, q4.w};
                    float hh[4], ll[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        hh[x] = __half2float(__float2half_rn(qq[x]));
                        ll[x] = qq[x] - hh[x];
                    }
                    const bool on = r < G;
                    qf[s2][0] = on ? pack_h2x(hh[0], hh[1]) : 0u;
                    qf[s2][2] = on ? pack_h2x(hh[2], hh[3]) : 0u;
                    qf[s2][1] = on ? pack_h2x(ll[0], ll[1]) : 0u;
                    qf[s2][3] = on ? pack_h2x(ll[2], ll[3]) : 0u;
                }
            }
            // S = Q C~^T on the tensor cores, n-tile by n-tile (8 candidates each);
            // thread (r, c) holds head r's scores of candidates 8 nt + 2c, + 1
            const uint32_t stg = ring_s + (it % NSTG) * STG;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const uint32_t row = 8 * nt + r;
                const uint32_t loc = __shfl_sync(0xffffffffu, d.local, row);
                float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int w2 = 0; w2 < KSF / 2; ++w2) {
                    uint4 kv;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                                 : "=r"(kv.x), "=r"(kv.y), "=r"(kv.z), "=r"(kv.w)
                                 : "r"(stg + row * ROWB + swz16(loc, c * (KSF / 2) + w2, D) * 16u));
                    mma_f16x(sc, qf[2 * w2], kv.x, kv.y);
                    mma_f16x(sd, qf[2 * w2 + 1], kv.z, kv.w);
                }
                if (r < G) {
                    s_sco[warp][r][8 * nt + 2 * c] = (sc[0] + sd[0]) + (sc[2] + sd[2]);
                    s_sco[warp][r][8 * nt + 2 * c + 1] = (sc[1] + sd[1]) + (sc[3] + sd[3]);
                }
            }
            } else {
            // small head dims: fp32 FMA per lane over its own row (c~ from shared memory)
            const uint32_t rowp = ring_s + (it % NSTG) * STG + lane * ROWB;
            float s4[GQ][4];
#pragma unroll
            for (int g = 0; g < GQ; ++g)
#pragma unroll
                for (int t = 0; t < 4; ++t) s4[g][t] = 0.f;
#pragma unroll
            for (uint32_t j2 = 0; j2 < V / 2; ++j2) {
                uint4 v16 = make_uint4(0u, 0u, 0u, 0u);
                if (d.valid)
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                                 : "=r"(v16.x), "=r"(v16.y), "=r"(v16.z), "=r"(v16.w)
                                 : "r"(rowp + swz16(d.local, j2, D) * 16u));
#pragma unroll
                for (uint32_t h2 = 0; h2 < 2; ++h2) {
                    const uint32_t j = 2 * j2 + h2;
                    const uint32_t w0 = h2 ? v16.z : v16.x, w1 = h2 ? v16.w : v16.y;
                    const float2 lo2 = __half22float2(*reinterpret_cast<const __half2*>(&w0));
                    const float2 hi2 = __half22float2(*reinterpret_cast<const __half2*>(&w1));
#pragma unroll
                    for (int g = 0; g < GQ; ++g) {
                        const float4 q4 = reinterpret_cast<const float4*>(qs + g * D)[j];
                        s4[g][0] = fmaf(q4.x, lo2.x, s4[g][0]);
                        s4[g][1] = fmaf(q4.y, lo2.y, s4[g][1]);
                        s4[g][2] = fmaf(q4.z, hi2.x, s4[g][2]);
                        s4[g][3] = fmaf(q4.w, hi2.y, s4[g][3]);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < GQ; ++g) s_sco[warp][g][lane] = (s4[g][0] + s4[g][1]) + (s4[g][2] + s4[g][3]);
            }
            __syncwarp();
            // the enclosure, per candidate on its own lane (k_select's bound, norm bound from fmeta)
            if (d.slot != mslot) {
                flush_minmax();
                mslot = d.slot;
#pragma unroll
                for (int g = 0; g < GQ; ++g) {
                    wmin[g] = ~0ull;
                    wmax[g] = 0ull;
                }
            }
            const PlanView pv(a.plan + (size_t)d.slot * a.plan_bytes, a);
            unsigned char* sc8 = p.scratch + (size_t)d.slot * G * p.qcap * kScratchEntry;
            unsigned long long* keys = reinterpret_cast<unsigned long long*>(sc8);
            uint32_t* wts = reinterpret_cast<uint32_t*>(keys + (size_t)G * p.qcap);
            double* his = reinterpret_cast<double*>(wts + (size_t)G * p.qcap);
            uint4 mt = make_uint4(0u, 0u, 0u, 0u);
            if (d.valid)
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(mt.x), "=r"(mt.y), "=r"(mt.z), "=r"(mt.w)
                             : "r"(meta_s + (it % NSTG) * MSTG + lane * 16u));
            const double rad = __hiloint2double((int)mt.y, (int)mt.x);
            const double cn = (double)__uint_as_float(mt.z);
            const uint32_t wt = p.mode == 1 ? mt.w : 1u;
#pragma unroll
            for (int g = 0; g < GQ; ++g) {
                if ((d.mask >> g) & 1u) {
                    const double qn = __ldg(pv.qnorm() + g);
                    const double ub = __dadd_rn((double)s_sco[warp][g][lane], __dmul_rn(qn, rad));
                    const double e = (qn * kFiK1 * cn + qn * kFiK2 + kFiK2 * cn +
                                      (fabs(ub) * kFiK3 + qn * kFiK3 * (cn + rad))) * (1.0 + 1e-9) + 1e-300;
                    const unsigned long long key = desc_key(ub - e);
                    const size_t at = (size_t)g * p.qcap + d.qoff[g] + d.local;
                    keys[at] = key;
                    wts[at] = wt;
                    his[at] = ub + e;
                    wmin[g] = min(wmin[g], key);
                    wmax[g] = max(wmax[g], key);
                }
            }
            __syncwarp();  // the stage is refilled two iterations later
            d = n1;
            n1 = n2;
            n2 = nb;
        }
        flush_minmax();
    }
    // the last CTA out resets the pool for the next launch
    __threadfence();
    __syncthreads();
    if (tid == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
        ctr[0] = 0;
        ctr[1] = 0;
    }
}

// ---------------------------------------------------------------------------
constexpr int kPkThreads = 256;
constexpr int kPkWarps = kPkThreads / 32;
constexpr uint32_t kPickStageTotal = 512;
  // selected clusters ranked from shared memory (all heads)

template <typename T>
__device__ __forceinline__ T pk_scan(T v, T* wt, T& total) {
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
        T t = lane < kPkWarps ? wt[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kPkWarps) wt[lane] = t;
    }
    __syncthreads();
    const T base = warp > 0 ? wt[warp - 1] : T(0);
    total = wt[kPkWarps - 1];
    __syncthreads();
    return base + x - v;
}

// k_pickq: one CTA per query head (128 threads).  Dynamic smem:
//   keys u64 [kPickKeysCap], weights / selection u32 [kPickKeysCap] (staged),
//   cbits u32 [words(cap_chunks)] this head's active-chunk bitmap.
constexpr int kPqThreads = 512;
constexpr int kPqWarps = kPqThreads / 32;

template <int DQ, int GQ>
__device__ __forceinline__ void pick_head(const Sel3Params& p) {
    constexpr uint32_t D = DQ;
    extern __shared__ __align__(16) unsigned char qsm[];
    const Arena& a = p.a;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t G = GQ;
    uint32_t g, slot;
    {  // this CTA's head: rank blockIdx in the size-class order k_coarse filed
        __shared__ uint32_t s_h;
        const uint32_t nh = gridDim.x * gridDim.y, b = blockIdx.y * gridDim.x + blockIdx.x;
        if (warp == 0) {
            const uint32_t cnt = lane < kPickClasses ? __ldcg(p.fine_ctr + 16 + lane) : 0u;
            uint32_t x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
            const unsigned int in = __ballot_sync(0xffffffffu, lane < kPickClasses && b < x);
            const uint32_t c = in ? (uint32_t)(__ffs(in) - 1) : 0u;
            const uint32_t before = __shfl_sync(0xffffffffu, x - cnt, c);
            if (lane == 0) {
                uint32_t h = b;  // identity if the filing is incomplete (never expected)
                if (total == nh && in) h = __ldcg(p.pick_ord + (size_t)c * nh + (b - before));
                s_h = h;
            }
        }
        __syncthreads();
        g = s_h % G;
        slot = a.slot0 + s_h / G;
    }
    const SlotState st = a.state[slot];
    const uint32_t M = st.n_chunks, P = st.P, L = st.L;
    PlanView pv(a.plan + (size_t)slot * a.plan_bytes, a);
    QInfo* qi = a.qinfo + (size_t)slot * G + g;
    if (pv.hdr()[0]) return;  // degenerate slot: build_spans writes everything
    LC_PMARK(0)
    const uint32_t mwcap = bit_words(a.cap_chunks), mw = bit_words(M);
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(qsm);
    uint32_t* sw = reinterpret_cast<uint32_t*>(sk + p.keys_cap);
    uint32_t* cb = sw + p.keys_cap;
    __shared__ uint32_t s_gbase[kMaxKU3], s_gpre[kMaxKU3 + 1], s_nc, s_kU;
    __shared__ __align__(16) unsigned char s_ph[PickPhase<DQ>::bytes];
    uint32_t* hw = reinterpret_cast<uint32_t*>(s_ph);  // radix histograms (weights, counts)
    uint32_t* hc = hw + 256;
    __shared__ unsigned long long s_prefix, s_mask, s_wbefore;
    __shared__ uint32_t s_cbefore, s_state, s_nsel;
    __shared__ int s_shift;
    constexpr uint32_t kStage = kPickStage;
    unsigned long long* s_sk = reinterpret_cast<unsigned long long*>(s_ph);
    uint32_t* s_sc = reinterpret_cast<uint32_t*>(s_ph + kStage * 8);
    uint32_t* s_so = reinterpret_cast<uint32_t*>(s_ph + kStage * 12);
    __shared__ double s_qd[DQ];  // q (f64) for the refinement's exact chains
    for (uint32_t j = tid; j < D; j += blockDim.x) s_qd[j] = (double)p.q[((size_t)slot * G + g) * D + j];
    for (uint32_t w = tid; w < mw; w += blockDim.x) cb[w] = 0u;
    if (warp == 0) {  // this head's kept units, in union order (ballot compaction)
        const uint32_t nuu = pv.hdr()[1];
        const uint32_t* uu = pv.units();
        uint32_t k2 = 0;
        for (uint32_t k0 = 0; k0 < nuu; k0 += 32) {
            const uint32_t k = k0 + lane;
            const bool mine = k < nuu && ((uu[k * (4 + G) + 1] >> g) & 1u);
            const unsigned int bal = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                const uint32_t at = k2 + __popc(bal & ((1u << lane) - 1u));
                s_gbase[at] = uu[k * (4 + G) + 2];
                s_gpre[at] = uu[k * (4 + G) + 4 + g];
            }
            k2 += __popc(bal);
        }
        if (lane == 0) s_gpre[k2] = pv.hdr()[4 + g];
    } else if (warp == 1 && lane == 0) {  // the plan header and key range, alongside warp 0's loads
        s_nc = pv.hdr()[4 + g];
        s_kU = pv.hdr()[3];
        const unsigned long long mn = pv.kmin()[g], mx = pv.kmax()[g];
        const unsigned long long diff = mn ^ mx;
        const int top = diff ? 63 - __clzll((long long)diff) : 0;
        const int shift = top >= 7 ? top - 7 : 0;  // first digit: the 8 highest differing bits
        const unsigned long long mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
        s_prefix = mn & mask;
        s_mask = mask;
        s_shift = shift;
        s_wbefore = 0;
        s_cbefore = 0;
        s_state = 0;
        s_nsel = 0;
    }
    __syncthreads();
    const uint32_t nc = s_nc, kU = s_kU;
    if (nc == 0 || nc > p.qcap) {
        if (tid == 0) {
            qi->error = nc == 0 ? kErrEmptyCand : kErrCandOverflow;
            qi->degenerate = 0;
            qi->n_units = kU;
            qi->n_clusters = 0;
            qi->scanned = P + nc;
            atomicOr(a.err, qi->error);
        }
        return;
    }
    unsigned long long* kg = reinterpret_cast<unsigned long long*>(p.scratch + (size_t)slot * G * p.qcap * kScratchEntry) +
                             (size_t)g * p.qcap;
    uint32_t* sg = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned long long*>(
                       p.scratch + (size_t)slot * G * p.qcap * kScratchEntry) + (size_t)G * p.qcap) + (size_t)g * p.qcap;
    // the filter's upper bounds, requested now: the refinement reads them after the select
    const double* hg = reinterpret_cast<const double*>(
                           p.scratch + (size_t)slot * G * p.qcap * kScratchEntry + (size_t)G * p.qcap * 12) +
                       (size_t)g * p.qcap;
    constexpr int kHPre = 8;
    const bool hpre_ok = nc <= kHPre * kPqThreads;
    double hpre[kHPre];
#pragma unroll
    for (int t = 0; t < kHPre; ++t) {
        const uint32_t i = t * kPqThreads + tid;
        hpre[t] = hpre_ok && i < nc ? hg[i] : -INFINITY;
    }
    if (nc <= p.keys_cap) {  // stage keys and weights (all loads in flight at once)
        for (uint32_t b0 = 0; b0 < nc; b0 += 8 * kPqThreads) {
            unsigned long long kv[8];
            uint32_t wv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t i = b0 + t * kPqThreads + tid;
                if (i < nc) {
                    kv[t] = kg[i];
                    wv[t] = sg[i];
                }
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t i = b0 + t * kPqThreads + tid;
                if (i < nc) {
                    sk[i] = kv[t];
                    sw[i] = wv[t];
                }
            }
        }
        kg = sk;
        sg = sw;
        __syncthreads();
    }
    LC_PMARK(1)
    auto cand = [&](uint32_t i) -> uint32_t {
        uint32_t k = 0;
        while (k + 1 < kU && s_gpre[k + 1] <= i) ++k;
        return s_gbase[k] + (i - s_gpre[k]);
    };
    const uint32_t* fo = a.forig + (size_t)slot * a.cap_clusters;
    const uint32_t* ft = a.ftok + (size_t)slot * a.cap_clusters;
    const uint32_t* moff_g = a.fmem_off + (size_t)slot * (a.cap_clusters + 1);
    const unsigned long long budget = p.mode == 1 ? p.budget : (unsigned long long)p.cluster_topk;
    // weighted radix select of the token-budget prefix (retriever.cpp:142-154):
    // the first key (ascending = descending score) at which the running weight
    // exceeds the budget.  Keys ~0 (candidates ruled out by the filter) are skipped.
    auto radix_select = [&]() {
    for (int shift = s_shift; shift >= 0; shift = shift >= 8 ? shift - 8 : (shift > 0 ? 0 : -1)) {
        for (uint32_t b = tid; b < 256; b += blockDim.x) {
            hw[b] = 0;
            hc[b] = 0;
        }
        __syncthreads();
        const unsigned long long prefix = s_prefix, mask = s_mask;
        for (uint32_t b0 = 0; b0 < nc; b0 += 4 * kPqThreads) {
            unsigned long long kv[4];
            uint32_t wv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t i = b0 + t * kPqThreads + tid;
                kv[t] = i < nc ? kg[i] : ~0ull;
                wv[t] = i < nc ? sg[i] : 0u;
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t i = b0 + t * kPqThreads + tid;
                if (i < nc && kv[t] != ~0ull && (kv[t] & mask) == prefix) {
                    atomicAdd(&hw[(uint32_t)(kv[t] >> shift) & 255u], wv[t]);
                    atomicAdd(&hc[(uint32_t)(kv[t] >> shift) & 255u], 1u);
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t w8[8], c8[8];
            unsigned long long lw = 0;
            uint32_t lc = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                w8[t] = hw[lane * 8 + t];
                c8[t] = hc[lane * 8 + t];
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
            unsigned long long cum = s_wbefore + (iw - lw), wexcl = 0;
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
                if (lane == 0) s_state = 2;
            } else if ((int)lane == __ffs(ballot) - 1) {
                const uint32_t b = lane * 8 + (uint32_t)found;
                s_prefix = prefix | ((unsigned long long)b << shift);
                s_mask = mask | (255ull << shift);
                s_wbefore = wexcl;
                s_cbefore += cexcl;
                s_state = c8[found] == 1 ? 1u : 0u;
            }
        }
        __syncthreads();
        if (s_state != 0) break;
    }
    };
    radix_select();  // on the filter's lower bounds (k_fine)
    LC_PMARK(2)
    // ---- exact refinement.  Let K* be the boundary key of the lower-bound walk
    // and x its score: the lower-bound prefix through K* weighs more than the
    // budget, so the exact walk overflows at or before score x, and every
    // cluster it admits (and the overflow one) has exact score >= x, hence upper
    // bound >= x.  Exact fp64 upper bounds (sequential chain, bit-exact
    // kernels::dot) for exactly those R = {hi >= x}; every other key becomes ~0.
    __shared__ uint32_t s_fast;
    {
        __shared__ unsigned long long s_xkey, s_rmin, s_rmax;
        __shared__ uint32_t s_rn;
        __shared__ uint32_t s_r[kPickRCap];
        if (tid == 0) {
            s_xkey = ~0ull;
            s_rmin = ~0ull;
            s_rmax = 0ull;
            s_rn = 0;
        }
        __syncthreads();
        const bool all = s_state == 2;
        if (!all) {
            const unsigned long long prefix = s_prefix, mask = s_mask;
            unsigned long long mn = ~0ull;
            for (uint32_t i = tid; i < nc; i += blockDim.x)
                if ((kg[i] & mask) == prefix) mn = min(mn, kg[i]);
            atomicMin(&s_xkey, mn);
        }
        __syncthreads();
        const double x = all ? -INFINITY : key_score(s_xkey);
        // R's arrays (fast path) follow the column slots in the phase buffer;
        // R's weights are read here, while the staged weights are live
        float4* s_col = reinterpret_cast<float4*>(s_ph);  // [kPickBufs * kPickCols][D / 4 + 1]
        unsigned long long* s_rk = reinterpret_cast<unsigned long long*>(s_ph + kPickBufs * kPickCols * (D + 4) * 4);
        double* s_rf = reinterpret_cast<double*>(s_rk + kPickRCap);
        uint32_t* s_ro = reinterpret_cast<uint32_t*>(s_rf + kPickRCap);
        uint32_t* s_rw = s_ro + kPickRCap;
        uint32_t* s_ri = s_rw + kPickRCap;
        uint32_t* s_rci = s_ri + kPickRCap;
        uint32_t* s_rmo = s_rci + kPickRCap;
        uint32_t* s_rmn = s_rmo + kPickRCap;
        // R as a list (ascending i) when it fits, else handled in place
        for (uint32_t b0 = 0; b0 < nc; b0 += 8 * kPqThreads) {  // eight loads in flight per thread
            double hv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t i = b0 + t * kPqThreads + tid;
                hv[t] = hpre_ok ? hpre[t] : (i < nc ? hg[i] : -INFINITY);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t i = b0 + t * kPqThreads + tid;
                if (i < nc && (all || hv[t] >= x)) {
                    const uint32_t at = atomicAdd(&s_rn, 1u);
                    if (at < kPickRCap) {
                        s_r[at] = i;
                        s_rw[at] = sg[i];
                    }
                }
            }
        }
        __syncthreads();
        const uint32_t nr = s_rn;
        if (p.prof && tid == 0) p.prof[((size_t)slot * GQ + g) * 8 + 7] = nr | ((unsigned long long)nc << 32);
        LC_PMARK(6)
        const float* fcs = a.fcent + (size_t)slot * a.cap_clusters * D;
        const double qn = pv.qnorm()[g];
        auto exact_key = [&](uint32_t i) -> unsigned long long {
            uint32_t k = 0;
            while (k + 1 < kU && s_gpre[k + 1] <= i) ++k;
            const uint32_t local = i - s_gpre[k], nu = s_gpre[k + 1] - s_gpre[k], ci = s_gbase[k] + local;
            const float4* col = reinterpret_cast<const float4*>(fcs + ((size_t)s_gbase[k] + local) * D);
            double sacc = 0.0;
            constexpr uint32_t B = D / 4 < 8 ? D / 4 : 8;  // rows per batch (head dims 8 / 16 have fewer)
            for (uint32_t j0 = 0; j0 < D / 4; j0 += B) {  // B loads in flight, then their chain steps
                float4 v4[B];
#pragma unroll
                for (uint32_t t = 0; t < B; ++t) v4[t] = __ldg(col + j0 + t);
#pragma unroll
                for (uint32_t t = 0; t < B; ++t) {
                const uint32_t jq = j0 + t;
                const float4 v = v4[t];
                sacc = __fma_rn(s_qd[4 * jq + 0], (double)v.x, sacc);
                sacc = __fma_rn(s_qd[4 * jq + 1], (double)v.y, sacc);
                sacc = __fma_rn(s_qd[4 * jq + 2], (double)v.z, sacc);
                sacc = __fma_rn(s_qd[4 * jq + 3], (double)v.w, sacc);
                }
            }
            return desc_key(__dadd_rn(sacc, __dmul_rn(qn, a.frad[(size_t)slot * a.cap_clusters + ci])));
        };
        unsigned long long rmn = ~0ull, rmx = 0ull;
        if (nr <= kPickRCap) {
            // R fits: select straight from it.  Rank R by (exact score desc,
            // reference id asc) -- select_topk's order (retriever.cpp:27-39) --
            // and admit the rank prefix while the running weight stays within
            // the budget, the first cluster unconditionally (retriever.cpp:142-154).
            // centroid columns of R by cp.async into column slots: the static
            // buffer, plus the staged keys / weights region once R's own fields
            // are read (nothing after this point reads it) -- usually all of R
            // in one round
            // (slots are D/4 + 1 float4s apart: the chains' column reads spread over the banks)
            const uint32_t nst = kPickBufs * kPickCols;
            const uint32_t nslots = nst + (uint32_t)((p.keys_cap * 12u) / (D * 4u + 16u));
            auto slot_col = [&](uint32_t k) -> float4* {
                return k < nst ? s_col + (size_t)k * (D / 4 + 1)
                               : reinterpret_cast<float4*>(qsm) + (size_t)(k - nst) * (D / 4 + 1);
            };
            auto issue = [&](uint32_t r0, uint32_t r1, uint32_t k0) {  // R entries [r0, r1) into slots k0..
                for (uint32_t x = tid; x < (r1 - r0) * (D / 4); x += blockDim.x) {
                    const uint32_t i = s_r[r0 + x / (D / 4)], jq = x % (D / 4);
                    uint32_t k = 0;
                    while (k + 1 < kU && s_gpre[k + 1] <= i) ++k;
                    const uint32_t local = i - s_gpre[k], nu = s_gpre[k + 1] - s_gpre[k];
                    const float4* src = reinterpret_cast<const float4*>(fcs + ((size_t)s_gbase[k] + local) * D) + jq;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(slot_col(k0 + x / (D / 4)) + jq)),
                                 "l"(src));
                }
            };
            issue(0, min(nr, nslots), 0);  // the keys / weights region is dead: R's weights are in s_rw
            asm volatile("cp.async.commit_group;\n" ::);
            // every other per-cluster field R needs, in one round of independent loads
            for (uint32_t r = tid; r < nr; r += blockDim.x) {
                const uint32_t i = s_r[r], ci = cand(i);
                s_rci[r] = ci;
                s_ro[r] = fo[ci];
                s_rf[r] = a.frad[(size_t)slot * a.cap_clusters + ci];
                s_rmo[r] = moff_g[ci];
                s_rmn[r] = moff_g[ci + 1];
            }
            for (uint32_t base = 0; base < nr; base += nslots) {
                if (base > 0) {
                    issue(base, min(nr, base + nslots), 0);
                    asm volatile("cp.async.commit_group;\n" ::);
                }
                asm volatile("cp.async.wait_group 0;\n" ::);
                __syncthreads();
                const uint32_t cnt = min(nslots, nr - base);
                for (uint32_t t = tid; t < cnt; t += blockDim.x) {
                    const float4* col = slot_col(t);
                    double sacc = 0.0;
#pragma unroll 8
                    for (uint32_t jq = 0; jq < D / 4; ++jq) {
                        const float4 v = col[jq];
                        sacc = __fma_rn(s_qd[4 * jq + 0], (double)v.x, sacc);
                        sacc = __fma_rn(s_qd[4 * jq + 1], (double)v.y, sacc);
                        sacc = __fma_rn(s_qd[4 * jq + 2], (double)v.z, sacc);
                        sacc = __fma_rn(s_qd[4 * jq + 3], (double)v.w, sacc);
                    }
                    s_rk[base + t] = desc_key(__dadd_rn(sacc, __dmul_rn(qn, s_rf[base + t])));
                }
                __syncthreads();  // the slots are free again
            }
            for (uint32_t r = tid; r < nr; r += blockDim.x) {
                const unsigned long long kr = s_rk[r];
                const uint32_t orr = s_ro[r];
                uint32_t rank = 0;
                for (uint32_t y = 0; y < nr; ++y) {
                    const unsigned long long ky = s_rk[y];
                    rank += (ky < kr || (ky == kr && s_ro[y] < orr)) ? 1u : 0u;
                }
                s_ri[rank] = r;
            }
            __syncthreads();
            if (warp == 0) {  // walk the ranks: running weight, first overflow ends the prefix
                unsigned long long run = 0;
                uint32_t nsel = nr;
                for (uint32_t b = 0; b < nr; b += 32) {
                    const uint32_t r = b + lane;
                    unsigned long long x = r < nr ? (unsigned long long)s_rw[s_ri[r]] : 0ull;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= (uint32_t)o) x += y;
                    }
                    const bool over = r < nr && r > 0 && run + x > budget;
                    const unsigned int bal = __ballot_sync(0xffffffffu, over);
                    if (bal) {
                        nsel = b + __ffs(bal) - 1;
                        break;
                    }
                    run += __shfl_sync(0xffffffffu, x, 31);
                }
                if (lane == 0) s_nsel = nsel;
            }
            if (tid == 0) s_fast = 1;
        } else {
            if (tid == 0) s_fast = 0;
            // large R (e.g. everything fits the budget): in place, one candidate per thread
            __syncthreads();
            for (uint32_t i = tid; i < nc; i += blockDim.x) {
                const bool in = all || hg[i] >= x;
                const unsigned long long k = in ? exact_key(i) : ~0ull;
                kg[i] = k;
                if (in) {
                    rmn = min(rmn, k);
                    rmx = max(rmx, k);
                }
            }
        }
        atomicMin(&s_rmin, rmn);
        atomicMax(&s_rmax, rmx);
        __syncthreads();
        if (tid == 0 && !s_fast) {
            const unsigned long long mn = s_rmin, mx = s_rmax;
            const unsigned long long diff = mn ^ mx;
            const int top = diff ? 63 - __clzll((long long)diff) : 0;
            const int shift = top >= 7 ? top - 7 : 0;  // first digit: the 8 highest differing bits
            const unsigned long long mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
            s_prefix = mn & mask;
            s_mask = mask;
            s_shift = shift;
            s_wbefore = 0;
            s_cbefore = 0;
            s_state = 0;
        }
        __syncthreads();
    }
    if (!s_fast) {
    radix_select();  // exact keys of R
    const unsigned long long prefix = s_prefix, mask = s_mask;
    const uint32_t state = s_state, cbefore = s_cbefore;
    for (uint32_t base = 0; base < nc; base += blockDim.x) {
        const uint32_t i = base + tid;
        bool take = false;
        if (i < nc && kg[i] != ~0ull) {
            const unsigned long long k = kg[i] & mask;
            take = k < prefix || (k == prefix && (state == 2 || (state == 1 && cbefore == 0)));
        }
        const unsigned int bal = __ballot_sync(0xffffffffu, take);
        uint32_t pos = 0;
        if (lane == 0 && bal) pos = atomicAdd(&s_nsel, (uint32_t)__popc(bal));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        __syncthreads();  // the list overwrites weights that other threads may still read
        if (take) sg[pos + __popc(bal & ((1u << lane) - 1u))] = i;
        __syncthreads();
    }
    if (state == 0 && tid == 0) {  // identical fp64 scores: reference-id order (retriever.cpp:33)
        unsigned long long used = s_wbefore;
        uint32_t admitted = cbefore, last_id = 0;
        bool first = true;
        for (;;) {
            int best = -1;
            uint32_t best_id = 0xffffffffu;
            for (uint32_t i = 0; i < nc; ++i) {
                if (kg[i] == ~0ull || (kg[i] & mask) != prefix) continue;
                const uint32_t oid = fo[cand(i)];
                if ((first || oid > last_id) && oid < best_id) {
                    best_id = oid;
                    best = (int)i;
                }
            }
            if (best < 0) break;
            const unsigned long long w = p.mode == 1 ? ft[cand((uint32_t)best)] : 1ull;
            if (admitted > 0 && used + w > budget) break;
            used += w;
            ++admitted;
            sg[s_nsel++] = (uint32_t)best;
            last_id = best_id;
            first = false;
        }
    }
    }
    __syncthreads();
    LC_PMARK(3)
    // rank order (select_topk order) + cluster bitmap + member chunks
    const uint32_t nsel = s_nsel;
    const bool fast = s_fast != 0;  // R's arrays (rank order, ids, member ranges) are still in s_ph
    const bool staged = !fast && nsel <= kStage;
    if (staged) {
        for (uint32_t x = tid; x < nsel; x += blockDim.x) {
            const uint32_t i = sg[x], ci = cand(i);
            s_sk[x] = kg[i];
            s_sc[x] = ci;
            s_so[x] = fo[ci];
        }
        __syncthreads();
    }
    uint32_t* out_cl = a.sel_clusters + ((size_t)slot * G + g) * a.cap_clusters;
    uint32_t* gbits = a.sel_bits + ((size_t)slot * G + g) * bit_words(a.cap_clusters);
    for (uint32_t w = tid; w < bit_words(L); w += blockDim.x) gbits[w] = 0u;
    __syncthreads();
    const uint32_t* moff = moff_g;
    const uint32_t* mem = a.fmem + (size_t)slot * a.cap_chunks;
    if (fast) {
        // the walk's rank order is select_topk's order; one warp per cluster
        // spreads its member chunks over the lanes
        const unsigned long long* s_rk = reinterpret_cast<const unsigned long long*>(s_ph + kPickBufs * kPickCols * (D + 4) * 4);
        const uint32_t* s_ro = reinterpret_cast<const uint32_t*>(s_rk + 2 * kPickRCap);
        const uint32_t* s_ri = s_ro + 2 * kPickRCap;
        const uint32_t* s_rci = s_ri + kPickRCap;
        const uint32_t* s_rmo = s_rci + kPickRCap;
        const uint32_t* s_rmn = s_rmo + kPickRCap;
        for (uint32_t x = warp; x < nsel; x += kPqWarps) {
            const uint32_t r = s_ri[x], ci = s_rci[r];
            if (lane == 0) {
                out_cl[x] = s_ro[r];
                atomicOr(&gbits[ci >> 5], 1u << (ci & 31));
            }
            for (uint32_t t = s_rmo[r] + lane; t < s_rmn[r]; t += 32) {
                const uint32_t j = mem[t];
                atomicOr(&cb[j >> 5], 1u << (j & 31));
            }
        }
    } else
    for (uint32_t x = tid; x < nsel; x += blockDim.x) {
        unsigned long long ki;
        uint32_t ci, oi, rank = 0;
        if (staged) {
            ki = s_sk[x];
            ci = s_sc[x];
            oi = s_so[x];
            for (uint32_t y = 0; y < nsel; ++y) {
                const unsigned long long ky = s_sk[y];
                rank += (ky < ki || (ky == ki && s_so[y] < oi)) ? 1u : 0u;
            }
        } else {
            const uint32_t i = sg[x];
            ki = kg[i];
            ci = cand(i);
            oi = fo[ci];
            for (uint32_t y = 0; y < nsel; ++y) {
                const unsigned long long ky = kg[sg[y]];
                if (ky < ki) ++rank;
                else if (ky == ki && y != x && fo[cand(sg[y])] < oi) ++rank;
            }
        }
        out_cl[rank] = oi;
        atomicOr(&gbits[ci >> 5], 1u << (ci & 31));
        for (uint32_t t = moff[ci]; t < moff[ci + 1]; ++t) {
            const uint32_t j = mem[t];
            atomicOr(&cb[j >> 5], 1u << (j & 31));
        }
    }
    __syncthreads();
    // grafted chunks [m0, M) are not in the member CSR: test their clusters
    if (st.m0 < M) {
        const uint32_t* cc = a.chunk_clu + (size_t)slot * a.cap_chunks;
        for (uint32_t j = st.m0 + tid; j < M; j += blockDim.x) {
            const uint32_t c = cc[j];
            if ((gbits[c >> 5] >> (c & 31)) & 1u) atomicOr(&cb[j >> 5], 1u << (j & 31));
        }
        __syncthreads();
    }
    LC_PMARK(4)
    uint32_t* gcb = a.chunk_bits + ((size_t)slot * G + g) * mwcap;
    for (uint32_t w = tid; w < mw; w += blockDim.x) gcb[w] = cb[w];
    if (tid == 0) {
        qi->n_units = kU;
        qi->n_clusters = nsel;
        qi->degenerate = 0;
        qi->error = 0;
        qi->scanned = (unsigned long long)P + nc;
    }
    LC_PMARK(5)
}

// build_spans: for one slot, by the last of its heads' k_pickq CTAs: union
// active spans in chunk order with per-head
// masks (collect_active, retriever.cpp:60-74), sink and buffer spans, counts.
constexpr int kSpMaxWarps = 8;
constexpr int kSpThreads = 256;
constexpr int kSpThreadsMax = kSpThreads;
constexpr uint32_t kSpCache = 1024;  // chunk spans kept in shared memory for the row-list pass

template <typename T>
__device__ __forceinline__ T sp_scan(T v, T* wt, T& total) {
    const int kSpWarps = (int)(blockDim.x >> 5);
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
        T t = lane < kSpWarps ? wt[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kSpWarps) wt[lane] = t;
    }
    __syncthreads();
    const T base = warp > 0 ? wt[warp - 1] : T(0);
    total = wt[kSpWarps - 1];
    __syncthreads();
    return base + x - v;
}

template <int GQ>
#define LC_SMARK(ph) \
    if (p.prof_sp && threadIdx.x == 0) p.prof_sp[(size_t)slot * 8 + (ph)] = gtime3();
__device__ __forceinline__ void build_spans(const Sel3Params& p, uint32_t slot) {
    LC_SMARK(0)
    const Arena& a = p.a;
    const uint32_t tid = threadIdx.x, lane = tid & 31, kSpWarps = blockDim.x >> 5;
    constexpr uint32_t G = GQ;
    const SlotState st = a.state[slot];
    const uint32_t n = st.n_tokens, M = st.n_chunks, ce = st.chunked_end, P = st.P, L = st.L;
    const uint32_t all = (1u << G) - 1u;
    PlanView pv(a.plan + (size_t)slot * a.plan_bytes, a);
    QInfo* qi = a.qinfo + (size_t)slot * G;
    Span* sp = a.spans + (size_t)slot * a.cap_spans;
    uint32_t* so = a.span_off + (size_t)slot * (a.cap_spans + 1);
    unsigned long long* sb = a.step_bytes + (size_t)slot * 4;
    uint32_t* rows = a.rows + (size_t)slot * a.cap_tokens;
    const unsigned long long dd = a.d;
    if (pv.hdr()[0]) {  // degenerate (retriever.cpp:86-95): everything, full attention
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
        for (uint32_t t = tid; t < n; t += blockDim.x) rows[t] = t | (all << 24);
        return;
    }
    __shared__ unsigned long long wtot[kSpMaxWarps];
    __shared__ uint32_t s_cnt[GQ], s_nsp[GQ], s_err;
    __shared__ uint32_t s_sst[kSpCache], s_slm[kSpCache], s_soff[kSpCache];
    __shared__ uint32_t s_bnd[33][kSpThreadsMax];  // each thread's word: its chunks' bounds
    if (tid < G) {
        s_cnt[tid] = 0;
        s_nsp[tid] = 0;
    }
    if (tid == 0) {
        uint32_t e = 0;
        for (uint32_t g = 0; g < G; ++g) e |= __ldcg(&qi[g].error);  // written by the other heads' CTAs
        s_err = e;
    }
    __syncthreads();
    if (s_err) {
        if (tid == 0) {
            a.n_spans[slot] = 0;
            so[0] = 0;
            a.slot_tok[slot] = 0;
        }
        return;
    }
    const uint32_t mwcap = bit_words(a.cap_chunks), mw = bit_words(M);
    const uint32_t* cbg = a.chunk_bits + (size_t)slot * G * mwcap;
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
        for (uint32_t t = tid; t < sink_end; t += blockDim.x) rows[t] = t | (all << 24);
    }
    const uint32_t* cs = a.chunk_start + (size_t)slot * (a.cap_chunks + 1);
    uint32_t my_cnt[GQ], my_nsp[GQ];
#pragma unroll
    for (int g = 0; g < GQ; ++g) my_cnt[g] = my_nsp[g] = 0;
    LC_SMARK(1)
    // software pipeline over rounds of blockDim words: round r + 1's bounds and
    // round r + 2's bitmap words are requested while round r is counted and
    // written, so only the prologue waits on memory
    const uint32_t W = blockDim.x;
    auto words = [&](uint32_t w, uint32_t* x) {
#pragma unroll
        for (int g = 0; g < GQ; ++g) x[g] = w < mw ? __ldcg(cbg + g * mwcap + w) : 0u;
    };
    // the bounds of the word's set chunks (chunk b's start and end), one batch of
    // independent loads
    auto bounds = [&](uint32_t w, const uint32_t* x, uint32_t* bnd) {
        uint32_t any = 0;
#pragma unroll
        for (int g = 0; g < GQ; ++g) any |= x[g];
#pragma unroll
        for (int b = 0; b <= 32; ++b) {
            const bool need = (b < 32 && ((any >> b) & 1u)) || (b > 0 && ((any >> (b - 1)) & 1u));
            bnd[b] = need ? __ldg(cs + w * 32 + b) : 0u;
        }
    };
    uint32_t cw[GQ], nx[GQ], nb[33];
    words(tid, cw);
    bounds(tid, cw, nb);
    words(tid + W, nx);
    for (uint32_t w0 = 0; w0 < mw; w0 += W) {
        const uint32_t w = w0 + tid;
        uint32_t wg[GQ], any = 0;
        // round r's bounds, parked in the thread's own shared column so the
        // loops below visit only the set bits
#pragma unroll
        for (int b = 0; b <= 32; ++b) s_bnd[b][tid] = nb[b];
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
            wg[g] = cw[g];
            any |= wg[g];
            cw[g] = nx[g];
        }
        if (w0 + W < mw) {
            bounds(w + W, cw, nb);
            words(w + 2 * W, nx);
        }
        uint32_t cnt = 0, toks = 0;
        for (uint32_t bits = any; bits; bits &= bits - 1u) {
            const uint32_t b = __ffs(bits) - 1;
            const uint32_t s0 = max(s_bnd[b][tid], sink_end), e0 = s_bnd[b + 1][tid];
            if (s0 < e0) {
                ++cnt;
                toks += e0 - s0;
            }
        }
        unsigned long long total;
        const unsigned long long ex = sp_scan<unsigned long long>(((unsigned long long)cnt << 40) | toks, wtot, total);
        uint32_t pos = out + (uint32_t)(ex >> 40), tp = tok + (uint32_t)(ex & 0xffffffffffull);
        for (uint32_t bits = any; bits; bits &= bits - 1u) {
            const uint32_t b = __ffs(bits) - 1;
            const uint32_t s0 = max(s_bnd[b][tid], sink_end), e0 = s_bnd[b + 1][tid];
            if (s0 >= e0) continue;
            uint32_t m = 0;
#pragma unroll
            for (int g = 0; g < GQ; ++g)
                if ((wg[g] >> b) & 1u) {
                    m |= 1u << g;
                    my_cnt[g] += e0 - s0;
                    my_nsp[g] += 1;
                }
            if (pos < a.cap_spans) {
                sp[pos].start = s0;
                sp[pos].len_mask = ((e0 - s0) << 8) | m;
                so[pos] = tp;
            }
            if (pos < kSpCache) {
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
    for (int g = 0; g < GQ; ++g) {
        const uint32_t c1 = __reduce_add_sync(0xffffffffu, my_cnt[g]);
        const uint32_t c2 = __reduce_add_sync(0xffffffffu, my_nsp[g]);
        if (lane == 0) {
            atomicAdd(&s_cnt[g], c1);
            atomicAdd(&s_nsp[g], c2);
        }
    }
    const uint32_t n_chunk_spans = out - (sink_end > 0 ? 1u : 0u);
    __syncthreads();
    LC_SMARK(2)
    {  // row list of the chunk spans: one thread per span writes its rows
        const uint32_t first = sink_end > 0 ? 1u : 0u, lim = min(out, a.cap_spans);
        for (uint32_t k = first + tid; k < lim; k += blockDim.x) {
            uint32_t st, lm, off;
            if (k < kSpCache) {
                st = s_sst[k];
                lm = s_slm[k];
                off = s_soff[k];
            } else {
                st = sp[k].start;
                lm = sp[k].len_mask;
                off = so[k];
            }
            const uint32_t len = lm >> 8, hm = (lm & 0xffu) << 24;
            for (uint32_t t = 0; t < len; ++t) rows[off + t] = (st + t) | hm;
        }
    }
    LC_SMARK(3)
    if (p.flags == 1u) {  // buffer_ids = [chunked_end, n), disjoint from the chunks
        const uint32_t b0 = max(ce, sink_end);
        if (n > b0) {
            if (tid == 0 && out < a.cap_spans) {
                sp[out].start = b0;
                sp[out].len_mask = ((n - b0) << 8) | all;
                so[out] = tok;
            }
            for (uint32_t t = tid; t < n - b0; t += blockDim.x) rows[tok + t] = (b0 + t) | (all << 24);
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
                        uint32_t m = 0;
#pragma unroll
                        for (int g = 0; g < GQ; ++g) m |= ((__ldcg(cbg + g * mwcap + (l >> 5)) >> (l & 31)) & 1u) << g;
                        resid = all & ~m;
                    }
                }
            }
            unsigned long long total;
            const unsigned long long ex = sp_scan<unsigned long long>(resid ? ((1ull << 40) | 1ull) : 0ull, wtot, total);
            if (resid) {
                rows[tok + (uint32_t)(ex & 0xffffffffffull)] = id | (resid << 24);
                const uint32_t pos = out + (uint32_t)(ex >> 40);
                if (pos < a.cap_spans) {
                    sp[pos].start = id;
                    sp[pos].len_mask = (1u << 8) | resid;
                    so[pos] = tok + (uint32_t)(ex & 0xffffffffffull);
                }
#pragma unroll
                for (int g = 0; g < GQ; ++g)
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
        a.slot_tok[slot] = tok;
        const unsigned long long Pl = P;
        const uint32_t bufl = (p.flags == 1u && n > max(ce, sink_end)) ? n - max(ce, sink_end) : 0u;
        unsigned long long per_q = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const unsigned long long act = (unsigned long long)s_cnt[g] + sink_end + bufl;
            qi[g].n_active = act;
            per_q += Pl * (4 * dd + 8) + (__ldcg(&qi[g].scanned) - Pl) * (4 * dd + 16) +
                     (unsigned long long)s_nsp[g] * 8 + act * 2 * dd * 2 + 8 * dd;
        }
        const unsigned long long ncu = pv.hdr()[2];
        sb[0] = Pl * (4 * dd + 8) + ncu * (4 * dd + 16) + (unsigned long long)n_chunk_spans * 8 +
                (unsigned long long)tok * 2 * dd * 2 + G * 8 * dd;
        sb[1] = per_q;
        sb[2] = tok;
        sb[3] = ncu;
    }
    LC_SMARK(4)
}

// k_pickq: one CTA per (query head, slot); k_spans: one CTA per slot.
template <int DQ, int GQ>
__global__ void __launch_bounds__(kPqThreads) k_pickq(Sel3Params p) {
    pdl_wait();
    pick_head<DQ, GQ>(p);
}

template <int GQ>
__global__ void __launch_bounds__(kSpThreads) k_spans(Sel3Params p) {
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x < kPickClasses) p.fine_ctr[16 + threadIdx.x] = 0;  // k_pickq is done
    build_spans<GQ>(p, p.a.slot0 + blockIdx.x);
}

size_t select3_pick_smem(const Arena& a);

// The failing stage of the last launch_select3 (thread-local; the ABI appends
// it to the error message).
thread_local char g_select3_where[96];
static cudaError_t select3_fail(cudaError_t e, const char* what, size_t arg) {
    snprintf(g_select3_where, sizeof g_select3_where, "%s (%zu)", what, arg);
    cudaGetLastError();  // a failed launch must not leak into the next call's error check
    return e;
}

// ---------------------------------------------------------------------------
template <int D, int GQ>
static cudaError_t launch3_dg(const Sel3Params& p, uint32_t n_slots, uint32_t max_union, uint32_t pmax,
                              cudaStream_t stream) {
    const size_t co_smem = (size_t)GQ * D * 8 + (size_t)D * ((pmax + 3) & ~3u) * 4 + (size_t)GQ * pmax * 8 +
                           (size_t)pmax * 16 + 4;  // urad, unit_off, union mask
    // k_pickq stages up to keys_cap candidates per head in shared memory: the
    // floor of 1024, raised when the grid leaves fewer CTAs per SM (long
    // contexts over few slots), so the radix passes stay on chip
    Sel3Params pp = p;
    const size_t bw = (size_t)bit_words(p.a.cap_chunks) * 4;
    {
        static KernelCfg pk_attr;
        const DevProps dp = dev_props();
        const int sms = dp.sms, smem_sm = dp.smem_sm, smem_blk = dp.smem_blk;
        const size_t st_smem = static_smem_of(k_pickq<D, GQ>, pk_attr);
        const unsigned long long ctas = (unsigned long long)n_slots * GQ;
        const unsigned long long per_sm = std::max(1ull, (ctas + sms - 1) / sms);
        const long long avail = std::min<long long>((long long)smem_sm / (long long)per_sm - 1024, smem_blk) -
                                (long long)st_smem - (long long)bw;
        const unsigned long long cap = avail > 0 ? ((unsigned long long)avail / 12) & ~1ull : 0ull;
        // only when it at least doubles the floor: a near-full SM keeps its CTA count
        if (cap >= 2ull * p.keys_cap)
            pp.keys_cap = (uint32_t)std::min<unsigned long long>(p.a.max_cand, cap);
    }
    if (const char* ev = getenv("LC_PICK_KEYS_CAP"))  // tests: force the unstaged (L2) key path
        pp.keys_cap = std::min<uint32_t>(pp.keys_cap, (uint32_t)std::max(2, atoi(ev)) & ~1u);
    const size_t pk_smem = (size_t)pp.keys_cap * 12 + bw;
    static KernelCfg co_cfg, pk_cfg, fi_cfg;
    cudaError_t e1 = ensure_smem(k_coarse<D, GQ>, co_cfg, co_smem);
    if (e1 != cudaSuccess) return select3_fail(e1, "k_coarse smem opt-in", co_smem);
    e1 = ensure_smem(k_pickq<D, GQ>, pk_cfg, pk_smem);
    if (e1 != cudaSuccess) return select3_fail(e1, "k_pickq smem opt-in", pk_smem);
    k_coarse<D, GQ><<<n_slots, kCoThreads, co_smem, stream>>>(p);
    e1 = cudaGetLastError();
    if (e1 != cudaSuccess) return select3_fail(e1, "k_coarse launch", co_smem);
    // k_fine: each warp's 3-stage row + metadata ring, then (D < 32) its q buffer
    const size_t fi_smem = (size_t)kFiWarps * (3 * 32 * (D * 2 + 16) + (D < 32 ? (size_t)GQ * D * 4 : 0));
    const uint32_t fine_grid = persistent_grid(k_fine<D, GQ>, fi_cfg, kFiThreads, fi_smem);
    for (uint32_t s0 = 0; s0 < n_slots; s0 += kMaxAttendSlots) {
        Sel3Params q = p;
        q.a.slot0 = p.a.slot0 + s0;
        cudaError_t e = launch_pdl(k_fine<D, GQ>, dim3(fine_grid), dim3(kFiThreads), fi_smem, stream, q,
                                   std::min<uint32_t>(kMaxAttendSlots, n_slots - s0));
        if (e != cudaSuccess) return select3_fail(e, "k_fine launch", fine_grid);
    }
    cudaError_t e2 = launch_pdl(k_pickq<D, GQ>, dim3(GQ, n_slots), dim3(kPqThreads), pk_smem, stream, pp);
    if (e2 != cudaSuccess) return select3_fail(e2, "k_pickq launch", pk_smem);
    e2 = launch_pdl(k_spans<GQ>, dim3(n_slots), dim3(kSpThreads), 0, stream, p);
    if (e2 != cudaSuccess) return select3_fail(e2, "k_spans launch", 0);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch3_d(const Sel3Params& p, uint32_t n_slots, uint32_t max_union, uint32_t pmax,
                             cudaStream_t stream) {
    switch (p.a.G) {
        case 1: return launch3_dg<D, 1>(p, n_slots, max_union, pmax, stream);
        case 4: return launch3_dg<D, 4>(p, n_slots, max_union, pmax, stream);
        default:
            if constexpr (D >= 64) {
                if (p.a.G == 2) return launch3_dg<D, 2>(p, n_slots, max_union, pmax, stream);
                if (p.a.G == 8) return launch3_dg<D, 8>(p, n_slots, max_union, pmax, stream);
            }
            return cudaErrorInvalidValue;
    }
}

static uint32_t pick_keys_cap(const Arena& a) { return a.max_cand < 1024u ? a.max_cand : 1024u; }

size_t select3_pick_smem(const Arena& a) {
    return (size_t)pick_keys_cap(a) * 12 + (size_t)bit_words(a.cap_chunks) * 4;
}

cudaError_t launch_select3(const Arena& a, const float* q, uint32_t unit_topk, uint32_t mode, uint32_t cluster_topk,
                           unsigned long long budget, uint32_t sink, uint32_t flags, const uint32_t* buf_off,
                           const uint32_t* buf_ids, unsigned char* scratch, uint32_t qcap, uint32_t max_union,
                           uint32_t pmax, uint32_t n_slots, uint32_t* fine_ctr, uint32_t* pick_ord,
                           cudaStream_t stream, const float* q_in) {
    // LC_PROF=1 (diagnostics only): per-CTA timestamps, buffers per device
    static unsigned long long *prof_dev[kMaxDevices] = {}, *prof_sp_dev[kMaxDevices] = {};
    const int dev = current_device();
    unsigned long long*& prof = prof_dev[dev];
    unsigned long long*& prof_sp = prof_sp_dev[dev];
    if (getenv("LC_PROF") && !prof) {
        cudaMalloc(&prof, (size_t)a.n_slots * a.G * 8 * 8);
        cudaMalloc(&prof_sp, (size_t)a.n_slots * 8 * 8);
        cudaMemset(prof_sp, 0, (size_t)a.n_slots * 8 * 8);
    }
    g_select3_where[0] = 0;
    Sel3Params p{a, pick_keys_cap(a), q, q_in ? q_in : q, unit_topk, mode, cluster_topk, sink, flags, budget, buf_off, buf_ids, scratch, qcap, prof,
                 fine_ctr, pick_ord, prof_sp};
    cudaError_t e = a.d == 128 ? launch3_d<128>(p, n_slots, max_union, pmax, stream)
                  : a.d == 64  ? launch3_d<64>(p, n_slots, max_union, pmax, stream)
                  : a.d == 32  ? launch3_d<32>(p, n_slots, max_union, pmax, stream)
                  : a.d == 16  ? launch3_d<16>(p, n_slots, max_union, pmax, stream)
                  : a.d == 8   ? launch3_d<8>(p, n_slots, max_union, pmax, stream)
                               : cudaErrorInvalidValue;
    if (prof && e == cudaSuccess) {
        cudaStreamSynchronize(stream);
        std::vector<unsigned long long> t((size_t)a.n_slots * a.G * 8);
        cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<double> tot;
        double acc[5] = {0, 0, 0, 0, 0};
        unsigned long long t0 = ~0ull, t1 = 0;
        for (size_t r = (size_t)a.slot0 * a.G; r < (size_t)(a.slot0 + n_slots) * a.G; ++r) {
            const unsigned long long* x = &t[r * 8];
            for (int k = 0; k < 5; ++k) acc[k] += (double)(x[k + 1] - x[k]);
            tot.push_back((double)(x[5] - x[0]));
            t0 = x[0] < t0 ? x[0] : t0;
            t1 = x[5] > t1 ? x[5] : t1;
        }
        std::sort(tot.begin(), tot.end());
        const double nq = (double)tot.size();
        double rs = 0, ncs = 0;
        for (size_t r = (size_t)a.slot0 * a.G; r < (size_t)(a.slot0 + n_slots) * a.G; ++r) {
            rs += (double)(t[r * 8 + 7] & 0xffffffffull);
            ncs += (double)(t[r * 8 + 7] >> 32);
        }
        double pre = 0;
        for (size_t r = (size_t)a.slot0 * a.G; r < (size_t)(a.slot0 + n_slots) * a.G; ++r) pre += (double)(t[r * 8 + 6] - t[r * 8 + 2]);
        unsigned long long rmax = 0;
        double tmax = 0;
        for (size_t r = (size_t)a.slot0 * a.G; r < (size_t)(a.slot0 + n_slots) * a.G; ++r)
            if ((double)(t[r * 8 + 5] - t[r * 8 + 0]) > tmax) {
                tmax = (double)(t[r * 8 + 5] - t[r * 8 + 0]);
                rmax = t[r * 8 + 7];
            }
        fprintf(stderr, "[LC_PROF] k_pickq refine set %.1f of %.1f candidates per head; x + R list %.2f us of refine; "
                "slowest head: |R| %llu of %llu, %.1f us\n", rs / nq, ncs / nq, pre / nq / 1e3, rmax & 0xffffffffull,
                rmax >> 32, tmax / 1e3);
        {
            std::vector<unsigned long long> u((size_t)a.n_slots * 8);
            cudaMemcpy(u.data(), prof_sp, u.size() * 8, cudaMemcpyDeviceToHost);
            double ph[4] = {0, 0, 0, 0}, cnt = 0, mx = 0;
            unsigned long long s0 = ~0ull, s1 = 0;
            for (size_t r = a.slot0; r < (size_t)a.slot0 + n_slots; ++r) {
                const unsigned long long* x = &u[r * 8];
                if (!x[4] || !x[0]) continue;
                for (int k = 0; k < 4; ++k) ph[k] += (double)(x[k + 1] - x[k]);
                mx = std::max(mx, (double)(x[4] - x[0]));
                s0 = std::min(s0, x[0]);
                s1 = std::max(s1, x[4]);
                cnt += 1;
            }
            if (cnt > 0)
                fprintf(stderr, "[LC_PROF] k_spans per-CTA us: setup %.2f words %.2f rows %.2f buffer+stats %.2f | max %.2f | span %.1f us\n",
                        ph[0] / cnt / 1e3, ph[1] / cnt / 1e3, ph[2] / cnt / 1e3, ph[3] / cnt / 1e3, mx / 1e3, (s1 - s0) / 1e3);
        }
        fprintf(stderr, "[LC_PROF] k_pickq per-CTA us: stage %.2f radix(lo) %.2f refine+select %.2f rank+members %.2f out %.2f | "
                "dur p50 %.2f p99 %.2f max %.2f | first start->last end %.1f us\n",
                acc[0] / nq / 1e3, acc[1] / nq / 1e3, acc[2] / nq / 1e3, acc[3] / nq / 1e3, acc[4] / nq / 1e3,
                tot[tot.size() / 2] / 1e3, tot[(size_t)(tot.size() * 0.99)] / 1e3, tot.back() / 1e3, (t1 - t0) / 1e3);
    }
    return e;
}

}  // namespace lc
