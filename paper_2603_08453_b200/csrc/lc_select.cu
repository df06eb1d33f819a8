// Fused scoring + pruning + selection (north star item 2) and active-set
// construction.  k_select: one CTA per query head (slot, g); k_compact: one
// CTA per slot (all query heads of the GQA group at once).
//
// Exactness (bit-identical to the reference's fp64 CPU path):
//  * kernels::dot (kernels.cpp:13-17) is a sequential fp64 sum of exact
//    float*float products, so a per-thread sequential DFMA chain over j
//    reproduces it bit-for-bit; no warp-tree reduction of a dot is used.
//  * UB = dot + qnorm*r (kernels.cpp:155-159) is __dmul_rn then __dadd_rn
//    (the reference is compiled without FMA).
//  * select_topk orders by (score desc, id asc) (retriever.cpp:27-39); the
//    greedy token-budget fill is a prefix of that order that stops at the
//    first overflow and always admits one cluster (retriever.cpp:142-154).
//    We find that prefix with an exact weighted radix select over the
//    orderable 64-bit image of the fp64 score (starting below the bits every
//    candidate shares, stopping as soon as the boundary bucket holds one
//    candidate), resolve exact-score ties by reference id, and sort only the
//    (small) selected set.
#include "lc_common.cuh"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lc {

struct SelectParams {
    Arena a;
    const float* q;  // [slot][G][d]
    uint32_t unit_topk, mode, cluster_topk, sink;
    unsigned long long budget;
    unsigned long long* prof;  // optional phase timestamps [slot*G + g][8] (LC_PROF=1)
};

__device__ __forceinline__ unsigned long long gtime_q() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define LC_QMARK(ph) \
    if (p.prof && threadIdx.x == 0) p.prof[((size_t)slot * a.G + g) * 8 + (ph)] = gtime_q();

constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kMaxUnitTopk = 64;

__device__ __forceinline__ bool key_less(unsigned long long ka, uint32_t ia,
                                         unsigned long long kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Dynamic shared memory of k_select:
//   float  qs[D]
//   u64    ukey[cap_units]
//   area:  first the coarse centroids [D][Pp] (staged once, coalesced), then
//          u64 ckey[C] candidate keys (ascending key == descending UB) and
//          u32 cw[C] weights (token_count, or 1 in fixed-k mode), reused as the
//          selected-index list.  C = smem_cand; larger candidate sets live in
//          the per-query-head global scratch (L2 resident) instead.
template <int D>
__global__ void __launch_bounds__(kSelThreads) k_select(SelectParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Arena& a = p.a;
    const uint32_t slot = a.slot0 + blockIdx.y, g = blockIdx.x, tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t d = D, dq = D / 4;
    const SlotState st = a.state[slot];
    QInfo* qi = a.qinfo + (size_t)slot * a.G + g;
    uint32_t* bits = a.sel_bits + ((size_t)slot * a.G + g) * bit_words(a.cap_clusters);
    const uint32_t nwords = bit_words(st.L);

    // degeneracy (retriever.cpp:86-95): whole store fits the budget, or no chunks
    const bool degenerate =
        (p.mode == 1 && (unsigned long long)st.n_tokens <= p.budget) || st.n_chunks == 0;
    if (degenerate) {
        if (tid == 0) {
            qi->n_units = st.P;
            qi->n_clusters = st.L;
            qi->degenerate = 1;
            qi->error = 0;
            qi->scanned = 0;
        }
        return;
    }

    float* qs = reinterpret_cast<float*>(smem);
    unsigned long long* ukey = reinterpret_cast<unsigned long long*>(smem + D * 4);
    unsigned char* area = smem + D * 4 + (size_t)a.cap_units * 8;
    const uint32_t Pp = (st.P + 3) & ~3u;
    float* ucs = reinterpret_cast<float*>(area);  // staged coarse centroids [D][Pp]

    __shared__ double s_qnorm;
    __shared__ uint32_t s_kept[kMaxUnitTopk];
    __shared__ uint32_t s_pre[kMaxUnitTopk + 1];
    __shared__ uint32_t s_base[kMaxUnitTopk], s_nu[kMaxUnitTopk];
    __shared__ uint32_t hw[256], hc[256];
    __shared__ unsigned long long s_min[kSelWarps], s_max[kSelWarps];
    __shared__ unsigned long long s_prefix, s_mask, s_wbefore;
    __shared__ uint32_t s_cbefore, s_state, s_nsel;
    __shared__ int s_shift;

    LC_QMARK(0)
    const float* qg = p.q + ((size_t)slot * a.G + g) * d;
    for (uint32_t j = tid; j < d; j += blockDim.x) qs[j] = qg[j];
    for (uint32_t w = tid; w < nwords; w += blockDim.x) bits[w] = 0u;
    // stage the coarse tier [D][P] (dimension-major rows of cap_units floats)
    const float* uc = a.ucent + (size_t)slot * a.cap_units * d;
    const bool staged = (size_t)D * Pp * 4 <= (size_t)a.smem_cand * 12 && (a.cap_units & 3) == 0;
    if (staged) {  // batched: every thread issues all its loads before any store
        const uint32_t pq = Pp >> 2, n4 = D * pq;
        constexpr int kB = 8;
        for (uint32_t e0 = 0; e0 < n4; e0 += kB * kSelThreads) {
            float4 v[kB];
#pragma unroll
            for (int t = 0; t < kB; ++t) {
                const uint32_t e = e0 + t * kSelThreads + tid;
                if (e < n4) v[t] = __ldg(reinterpret_cast<const float4*>(uc + (size_t)(e / pq) * a.cap_units) + e % pq);
            }
#pragma unroll
            for (int t = 0; t < kB; ++t) {
                const uint32_t e = e0 + t * kSelThreads + tid;
                if (e < n4) reinterpret_cast<float4*>(ucs + (size_t)(e / pq) * Pp)[e % pq] = v[t];
            }
        }
    }
    __syncthreads();

    LC_QMARK(1)
    // ||q|| (kernels.cpp:19-23): sequential, exact products -> DFMA chain
    if (tid == 0) {
        double s = 0.0;
#pragma unroll 8
        for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)qs[j], (double)qs[j], s);
        s_qnorm = __dsqrt_rn(s);
    }
    // tier 1: coarse units (retriever.cpp:100-112); warp 0 is busy with ||q||
    const double* ur = a.urad + (size_t)slot * a.cap_units;
    double udot[5];
    const uint32_t ct = tid >= 32 ? tid - 32 : 0xffffffffu;
#pragma unroll
    for (uint32_t k = 0; k < 5; ++k) {
        const uint32_t u = ct + k * (kSelThreads - 32);
        double s = 0.0;
        if (ct != 0xffffffffu && u < st.P) {
            if (staged) {
#pragma unroll 8
                for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)qs[j], (double)ucs[j * Pp + u], s);
            } else {
                for (uint32_t j = 0; j < d; ++j)
                    s = __fma_rn((double)qs[j], (double)__ldg(uc + (size_t)j * a.cap_units + u), s);
            }
        }
        udot[k] = s;
    }
    __syncthreads();
    const double qnorm = s_qnorm;
#pragma unroll
    for (uint32_t k = 0; k < 5; ++k) {
        const uint32_t u = ct + k * (kSelThreads - 32);
        if (ct != 0xffffffffu && u < st.P) ukey[u] = desc_key(__dadd_rn(udot[k], __dmul_rn(qnorm, ur[u])));
    }
    __syncthreads();
    // select_topk(units, unit_topk): rank by counting over (score desc, id asc)
    const uint32_t kU = min(min(p.unit_topk, st.P), (uint32_t)kMaxUnitTopk);
    for (uint32_t u = tid; u < st.P; u += blockDim.x) {
        const unsigned long long ku = ukey[u];
        uint32_t rank = 0;
        for (uint32_t v = 0; v < st.P; ++v) rank += key_less(ukey[v], v, ku, u) ? 1u : 0u;
        if (rank < kU) s_kept[rank] = u;
    }
    __syncthreads();
    const uint32_t* uoff = a.unit_off + (size_t)slot * (a.cap_units + 1);
    if (tid == 0) {
        uint32_t acc = 0;
        for (uint32_t k = 0; k < kU; ++k) {
            s_pre[k] = acc;
            const uint32_t u = s_kept[k];
            s_base[k] = uoff[u];
            s_nu[k] = uoff[u + 1] - uoff[u];
            acc += s_nu[k];
        }
        s_pre[kU] = acc;
    }
    __syncthreads();
    const uint32_t nc = s_pre[kU];
    if (nc > a.max_cand || nc == 0 || (nc > a.smem_cand && a.cand_scratch == nullptr)) {
        if (tid == 0) {
            qi->error = nc == 0 ? kErrEmptyCand : kErrCandOverflow;
            qi->degenerate = 0;
            qi->n_units = kU;
            qi->n_clusters = 0;
            qi->scanned = st.P + nc;
            atomicOr(a.err, qi->error);
        }
        return;
    }
    // candidate storage: shared memory, or this query head's global scratch
    unsigned long long* ckey;
    uint32_t* cw;
    if (nc <= a.smem_cand) {
        ckey = reinterpret_cast<unsigned long long*>(area);
        cw = reinterpret_cast<uint32_t*>(ckey + a.smem_cand);
    } else {
        unsigned char* gs = a.cand_scratch + ((size_t)slot * a.G + g) * (size_t)a.max_cand * 12;
        ckey = reinterpret_cast<unsigned long long*>(gs);
        cw = reinterpret_cast<uint32_t*>(ckey + a.max_cand);
    }

    LC_QMARK(2)
    // tier 2: fine clusters of the kept units (retriever.cpp:118-135); the
    // unit blocks are [D/4][n_u][4]: one float4 per cluster per step, loads
    // double-buffered four quads ahead of the sequential DFMA chain
    const float* fc = a.fcent + (size_t)slot * a.cap_clusters * d;
    const double* fr = a.frad + (size_t)slot * a.cap_clusters;
    const uint32_t* ft = a.ftok + (size_t)slot * a.cap_clusters;
    unsigned long long kmin = ~0ull, kmax = 0ull;
    // two candidates per thread at a time: two independent DFMA chains and
    // twice the loads in flight
    auto locate = [&](uint32_t i, uint32_t& base, uint32_t& nu, uint32_t& local) {
        uint32_t k = 0;
        while (k + 1 < kU && s_pre[k + 1] <= i) ++k;
        base = s_base[k];
        nu = s_nu[k];
        local = i - s_pre[k];
    };
    for (uint32_t i0 = tid; i0 < nc; i0 += 2 * blockDim.x) {
        const uint32_t i1 = i0 + blockDim.x;
        const bool has1 = i1 < nc;
        uint32_t b0, n0, l0, b1 = 0, n1 = 1, l1 = 0;
        locate(i0, b0, n0, l0);
        if (has1) locate(i1, b1, n1, l1);
        const float4* c0 = reinterpret_cast<const float4*>(fc + (size_t)b0 * d) + l0;
        const float4* c1 = has1 ? reinterpret_cast<const float4*>(fc + (size_t)b1 * d) + l1 : c0;
        const uint32_t cid0 = b0 + l0, cid1 = has1 ? b1 + l1 : cid0;
        const double r0 = fr[cid0], r1 = fr[cid1];
        const uint32_t w0 = p.mode == 1 ? ft[cid0] : 1u, w1 = p.mode == 1 ? ft[cid1] : 1u;
        float4 A0[4], A1[4], B0[4], B1[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            A0[t] = __ldg(c0 + (size_t)t * n0);
            A1[t] = __ldg(c1 + (size_t)t * n1);
        }
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (uint32_t jq = 0; jq < dq; jq += 4) {
            if (jq + 4 < dq) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    B0[t] = __ldg(c0 + (size_t)(jq + 4 + t) * n0);
                    B1[t] = __ldg(c1 + (size_t)(jq + 4 + t) * n1);
                }
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float4 q4 = reinterpret_cast<const float4*>(qs)[jq + t];
                s0 = __fma_rn((double)q4.x, (double)A0[t].x, s0);
                s1 = __fma_rn((double)q4.x, (double)A1[t].x, s1);
                s0 = __fma_rn((double)q4.y, (double)A0[t].y, s0);
                s1 = __fma_rn((double)q4.y, (double)A1[t].y, s1);
                s0 = __fma_rn((double)q4.z, (double)A0[t].z, s0);
                s1 = __fma_rn((double)q4.z, (double)A1[t].z, s1);
                s0 = __fma_rn((double)q4.w, (double)A0[t].w, s0);
                s1 = __fma_rn((double)q4.w, (double)A1[t].w, s1);
            }
            if (jq + 4 < dq) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    A0[t] = B0[t];
                    A1[t] = B1[t];
                }
            }
        }
        const unsigned long long k0 = desc_key(__dadd_rn(s0, __dmul_rn(qnorm, r0)));
        ckey[i0] = k0;
        cw[i0] = w0;
        kmin = min(kmin, k0);
        kmax = max(kmax, k0);
        if (has1) {
            const unsigned long long k1 = desc_key(__dadd_rn(s1, __dmul_rn(qnorm, r1)));
            ckey[i1] = k1;
            cw[i1] = w1;
            kmin = min(kmin, k1);
            kmax = max(kmax, k1);
        }
    }
    // the bits every candidate shares are skipped by the radix passes
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
        s_min[warp] = kmin;
        s_max[warp] = kmax;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long mn = s_min[0], mx = s_max[0];
        for (int w = 1; w < kSelWarps; ++w) {
            mn = min(mn, s_min[w]);
            mx = max(mx, s_max[w]);
        }
        const unsigned long long diff = mn ^ mx;
        int top = diff ? 63 - __clzll((long long)diff) : 0;  // highest differing bit
        int shift = (top / 8) * 8;                           // byte holding it
        unsigned long long mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
        s_prefix = mn & mask;
        s_mask = mask;
        s_shift = shift;
        s_wbefore = 0;
        s_cbefore = 0;
        s_state = 0;
        s_nsel = 0;
    }
    __syncthreads();

    LC_QMARK(3)
    // weighted prefix select: the longest prefix of the (key, id) order whose
    // weight sum stays <= budget (retriever.cpp:146-153); fixed-k mode is the
    // same with unit weights and budget = k_c (select_topk, retriever.cpp:141)
    const unsigned long long budget = p.mode == 1 ? p.budget : (unsigned long long)p.cluster_topk;
    for (int shift = s_shift; shift >= 0; shift -= 8) {
        for (uint32_t b = tid; b < 256; b += blockDim.x) {
            hw[b] = 0;
            hc[b] = 0;
        }
        __syncthreads();
        const unsigned long long prefix = s_prefix, mask = s_mask;
        for (uint32_t i = tid; i < nc; i += blockDim.x) {
            const unsigned long long k = ckey[i];
            if ((k & mask) == prefix) {
                const uint32_t b = (uint32_t)(k >> shift) & 255u;
                atomicAdd(&hw[b], cw[i]);
                atomicAdd(&hc[b], 1u);
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
            const unsigned long long wbase = s_wbefore + (iw - lw);
            const uint32_t cbase = ic - lc;
            int found = -1;
            unsigned long long cum = wbase, wexcl = 0;
            uint32_t ccum = cbase, cexcl = 0;
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
                if (lane == 0) s_state = 2;  // everything matching fits
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
    // mark the selection (compacted into the weight array, no longer needed)
    const unsigned long long prefix = s_prefix, mask = s_mask;
    const uint32_t state = s_state;
    const uint32_t cbefore = s_cbefore;
    for (uint32_t base = 0; base < nc; base += blockDim.x) {
        const uint32_t i = base + tid;
        bool take = false;
        if (i < nc) {
            const unsigned long long k = ckey[i] & mask;
            take = k < prefix;
            if (k == prefix) {
                if (state == 2) take = true;                 // whole bucket fits
                else if (state == 1) take = cbefore == 0;    // lone boundary: admit if first
            }
        }
        const unsigned int bal = __ballot_sync(0xffffffffu, take);
        uint32_t pos = 0;
        if (lane == 0 && bal) pos = atomicAdd(&s_nsel, (uint32_t)__popc(bal));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (take) cw[pos + __popc(bal & ((1u << lane) - 1u))] = i;
    }
    __syncthreads();
    const uint32_t* fo = a.forig + (size_t)slot * a.cap_clusters;
    auto cid_of = [&](uint32_t i) -> uint32_t {
        uint32_t k = 0;
        while (k + 1 < kU && s_pre[k + 1] <= i) ++k;
        return s_base[k] + (i - s_pre[k]);
    };
    if (state == 0 && tid == 0) {
        // bucket of identical fp64 scores: reference-id order (retriever.cpp:33)
        unsigned long long used = s_wbefore;
        uint32_t admitted = cbefore;
        uint32_t last_id = 0;
        bool first = true;
        for (;;) {
            int best = -1;
            uint32_t best_id = 0xffffffffu;
            for (uint32_t i = 0; i < nc; ++i) {
                if ((ckey[i] & mask) != prefix) continue;
                const uint32_t oid = fo[cid_of(i)];
                if ((first || oid > last_id) && oid < best_id) {
                    best_id = oid;
                    best = (int)i;
                }
            }
            if (best < 0) break;
            const unsigned long long w = p.mode == 1 ? a.ftok[(size_t)slot * a.cap_clusters + cid_of(best)] : 1ull;
            if (admitted > 0 && used + w > budget) break;
            used += w;
            ++admitted;
            cw[s_nsel++] = (uint32_t)best;
            last_id = best_id;
            first = false;
        }
    }
    __syncthreads();

    LC_QMARK(4)
    // rank order of the selected set + outputs
    const uint32_t nsel = s_nsel;
    uint32_t* out_cl = a.sel_clusters + ((size_t)slot * a.G + g) * a.cap_clusters;
    for (uint32_t x = tid; x < nsel; x += blockDim.x) {
        const uint32_t i = cw[x];
        const unsigned long long ki = ckey[i];
        const uint32_t ci = cid_of(i);
        const uint32_t oi = fo[ci];
        uint32_t rank = 0;
        for (uint32_t y = 0; y < nsel; ++y) {
            const unsigned long long ky = ckey[cw[y]];
            if (ky < ki) ++rank;
            else if (ky == ki && y != x && fo[cid_of(cw[y])] < oi) ++rank;
        }
        out_cl[rank] = oi;
        atomicOr(&bits[ci >> 5], 1u << (ci & 31));
    }
    uint32_t* out_u = a.sel_units + ((size_t)slot * a.G + g) * a.cap_units;
    for (uint32_t k = tid; k < kU; k += blockDim.x) out_u[k] = s_kept[k];
    if (tid == 0) {
        qi->n_units = kU;
        qi->n_clusters = nsel;
        qi->degenerate = 0;
        qi->error = 0;
        qi->scanned = (unsigned long long)st.P + nc;
    }
    LC_QMARK(5)
}

// ---------------------------------------------------------------------------
// Active-set construction (collect_active, retriever.cpp:60-74) for every query
// head of a slot at once: one pass over the chunk table produces the union of
// the group's active chunk spans, each tagged with the mask of query heads it
// serves, in token order.  Sink [0, min(sink, n)) is emitted once for all heads
// and chunk spans are clipped against it, so the union has no duplicates.
struct CompactParams {
    Arena a;
    uint32_t sink, flags;
    const uint32_t* buf_off;  // LC_BUFFER_LIST
    const uint32_t* buf_ids;
};

constexpr int kCompactThreads = 512;
constexpr int kChunksPerThread = 8;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* warp_tot, T& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        T t = lane < nw ? warp_tot[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) warp_tot[lane] = t;
    }
    __syncthreads();
    const T base = warp > 0 ? warp_tot[warp - 1] : T(0);
    total = warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
    return base + x - v;
}

__global__ void __launch_bounds__(kCompactThreads) k_compact(CompactParams p) {
    extern __shared__ __align__(16) uint32_t sbits[];  // [G][words(L)] then u8 cmask[L]
    const Arena& a = p.a;
    const uint32_t slot = a.slot0 + blockIdx.x, tid = threadIdx.x, G = a.G, lane = tid & 31;
    const SlotState st = a.state[slot];
    const uint32_t n = st.n_tokens, M = st.n_chunks, ce = st.chunked_end;
    const uint32_t all = (1u << G) - 1u;
    Span* sp = a.spans + (size_t)slot * a.cap_spans;
    uint32_t* so = a.span_off + (size_t)slot * (a.cap_spans + 1);
    QInfo* qi = a.qinfo + (size_t)slot * G;
    unsigned long long* sb = a.step_bytes + (size_t)slot * 4;
    const unsigned long long d = a.d;

    __shared__ uint32_t s_cnt[kMaxGroup];
    __shared__ uint32_t s_nsp[kMaxGroup];
    __shared__ unsigned long long warp_tot[kCompactThreads / 32];
    __shared__ uint32_t s_units[32];  // union of kept units (bitset, cap_units <= 1024)

    if (qi[0].degenerate) {
        if (tid == 0) {
            sp[0].start = 0;
            sp[0].len_mask = (n << 8) | all;
            so[0] = 0;
            so[1] = n;
            a.n_spans[slot] = 1;
            for (uint32_t g = 0; g < G; ++g) qi[g].n_active = n;
            sb[0] = d * 2 * 2 * n + G * 8 * d;
            sb[1] = (d * 2 * 2 * n + 8 * d) * G;
            sb[2] = n;
            sb[3] = 0;
        }
        return;
    }
    const uint32_t words = bit_words(st.L);
    const uint32_t* gbits = a.sel_bits + (size_t)slot * G * bit_words(a.cap_clusters);
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t w = tid; w < words; w += blockDim.x)
            sbits[g * words + w] = gbits[(size_t)g * bit_words(a.cap_clusters) + w];
    if (tid < kMaxGroup) {
        s_cnt[tid] = 0;
        s_nsp[tid] = 0;
    }
    if (tid < 32) s_units[tid] = 0;
    __syncthreads();
    // per-cluster mask of the query heads that selected it
    uint8_t* cmask = reinterpret_cast<uint8_t*>(sbits + G * words);
    for (uint32_t c = tid; c < st.L; c += blockDim.x) {
        uint32_t m = 0;
        for (uint32_t g = 0; g < G; ++g) m |= ((sbits[g * words + (c >> 5)] >> (c & 31)) & 1u) << g;
        cmask[c] = (uint8_t)m;
    }
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
    uint32_t my_cnt[kMaxGroup], my_nsp[kMaxGroup];
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) my_cnt[g] = my_nsp[g] = 0;
    constexpr uint32_t kTile = kCompactThreads * kChunksPerThread;
    for (uint32_t base = 0; base < M; base += kTile) {
        const uint32_t j0 = base + tid * kChunksPerThread;
        uint32_t m8[kChunksPerThread], s8[kChunksPerThread], l8[kChunksPerThread];
        uint32_t cnt = 0, toks = 0;
        uint32_t cl[kChunksPerThread];
#pragma unroll
        for (int e = 0; e < kChunksPerThread; ++e) cl[e] = j0 + e < M ? __ldg(cc + j0 + e) : 0u;
#pragma unroll
        for (int e = 0; e < kChunksPerThread; ++e) m8[e] = j0 + e < M ? cmask[cl[e]] : 0u;
        uint32_t e8[kChunksPerThread];
#pragma unroll
        for (int e = 0; e < kChunksPerThread; ++e) {
            s8[e] = m8[e] ? __ldg(cs + j0 + e) : 0u;
            e8[e] = m8[e] ? __ldg(cs + j0 + e + 1) : 0u;
        }
#pragma unroll
        for (int e = 0; e < kChunksPerThread; ++e) {
            uint32_t m = m8[e], len = 0;
            if (m) {
                const uint32_t st0 = max(s8[e], sink_end);
                if (st0 >= e8[e]) {
                    m = 0;
                } else {
                    s8[e] = st0;
                    len = e8[e] - st0;
                    cnt += 1;
                    toks += len;
#pragma unroll
                    for (int g = 0; g < kMaxGroup; ++g)
                        if ((m >> g) & 1u) {
                            my_cnt[g] += len;
                            my_nsp[g] += 1;
                        }
                }
            }
            m8[e] = m;
            l8[e] = len;
        }
        const unsigned long long v = ((unsigned long long)cnt << 40) | toks;
        unsigned long long total;
        const unsigned long long ex = block_excl_scan(v, warp_tot, total);
        uint32_t pos = out + (uint32_t)(ex >> 40);
        uint32_t tp = tok + (uint32_t)(ex & 0xffffffffffull);
#pragma unroll
        for (int e = 0; e < kChunksPerThread; ++e) {
            if (m8[e]) {
                if (pos < a.cap_spans) {
                    sp[pos].start = s8[e];
                    sp[pos].len_mask = (l8[e] << 8) | m8[e];
                    so[pos] = tp;
                }
                ++pos;
                tp += l8[e];
            }
        }
        out += (uint32_t)(total >> 40);
        tok += (uint32_t)(total & 0xffffffffffull);
    }
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
        if ((uint32_t)g >= G) break;
        const uint32_t c1 = __reduce_add_sync(0xffffffffu, my_cnt[g]);
        const uint32_t c2 = __reduce_add_sync(0xffffffffu, my_nsp[g]);
        if (lane == 0) {
            atomicAdd(&s_cnt[g], c1);
            atomicAdd(&s_nsp[g], c2);
        }
    }
    const uint32_t n_chunk_spans = out - (sink_end > 0 ? 1u : 0u);
    // buffer ids (collect_active, retriever.cpp:71)
    if (p.flags == 1u) {  // LC_BUFFER_STREAM: [chunked_end, n), disjoint from chunks
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
                        uint32_t l = 0, h = M;  // last chunk with start <= id
                        while (h - l > 1) {
                            const uint32_t mid = (l + h) >> 1;
                            if (cs[mid] <= id) l = mid;
                            else h = mid;
                        }
                        const uint32_t c = cc[l];
                        uint32_t m = 0;
                        for (uint32_t g = 0; g < G; ++g)
                            m |= ((sbits[g * words + (c >> 5)] >> (c & 31)) & 1u) << g;
                        resid = all & ~m;
                    }
                }
            }
            const unsigned long long v = resid ? ((1ull << 40) | 1ull) : 0ull;
            unsigned long long total;
            const unsigned long long ex = block_excl_scan(v, warp_tot, total);
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
    // kept-unit union for the byte accounting
    const uint32_t* su = a.sel_units + (size_t)slot * G * a.cap_units;
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t k = tid; k < qi[g].n_units; k += blockDim.x) {
            const uint32_t u = su[(size_t)g * a.cap_units + k];
            if (u < 1024) atomicOr(&s_units[u >> 5], 1u << (u & 31));
        }
    __syncthreads();
    if (tid == 0) {
        if (out > a.cap_spans) {
            atomicOr(a.err, kErrSpanOverflow);
            out = a.cap_spans;
        }
        so[out] = tok;
        a.n_spans[slot] = out;
        const uint32_t* uoff = a.unit_off + (size_t)slot * (a.cap_units + 1);
        unsigned long long nc_union = 0;
        for (uint32_t u = 0; u < st.P && u < 1024; ++u)
            if ((s_units[u >> 5] >> (u & 31)) & 1u) nc_union += uoff[u + 1] - uoff[u];
        const unsigned long long P = st.P;
        unsigned long long per_q = 0;
        const uint32_t bufl = (p.flags == 1u && n > max(ce, sink_end)) ? n - max(ce, sink_end) : 0u;
        for (uint32_t g = 0; g < G; ++g) {
            const unsigned long long act = (unsigned long long)s_cnt[g] + sink_end + bufl;
            qi[g].n_active = act;
            const unsigned long long ncg = qi[g].scanned - P;
            per_q += P * (4 * d + 8) + ncg * (4 * d + 16) + (unsigned long long)s_nsp[g] * 8 +
                     act * 2 * d * 2 + 8 * d;
        }
        sb[0] = P * (4 * d + 8) + nc_union * (4 * d + 16) + (unsigned long long)n_chunk_spans * 8 +
                (unsigned long long)tok * 2 * d * 2 + G * 8 * d;
        sb[1] = per_q;
        sb[2] = tok;
        sb[3] = nc_union;
    }
}

// launchers ------------------------------------------------------------------
size_t select_smem_bytes(const Arena& a) {
    return (size_t)a.d * 4 + (size_t)a.cap_units * 8 + (size_t)a.smem_cand * 12;
}

template <int D>
static cudaError_t launch_select_d(const SelectParams& p, uint32_t n_slots, size_t smem, cudaStream_t stream) {
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(k_select<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    k_select<D><<<dim3(p.a.G, n_slots), kSelThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_select(const Arena& a, const float* q, uint32_t unit_topk, uint32_t mode,
                          uint32_t cluster_topk, unsigned long long budget, uint32_t sink,
                          uint32_t n_slots, cudaStream_t stream) {
    static unsigned long long* prof = nullptr;
    if (getenv("LC_PROF") && !prof) cudaMalloc(&prof, (size_t)a.n_slots * a.G * 8 * 8);
    SelectParams p{a, q, unit_topk, mode, cluster_topk, sink, budget, prof};
    const size_t smem = select_smem_bytes(a);
    cudaError_t e = a.d == 128 ? launch_select_d<128>(p, n_slots, smem, stream)
                  : a.d == 64  ? launch_select_d<64>(p, n_slots, smem, stream)
                               : cudaErrorInvalidValue;
    if (prof && e == cudaSuccess) {
        cudaStreamSynchronize(stream);
        std::vector<unsigned long long> t((size_t)a.n_slots * a.G * 8);
        cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
        double acc[5] = {0, 0, 0, 0, 0};
        unsigned long long t0 = ~0ull, t1 = 0;
        size_t cnt = 0;
        for (uint32_t s = a.slot0; s < a.slot0 + n_slots; ++s)
            for (uint32_t g = 0; g < a.G; ++g) {
                const unsigned long long* r = &t[((size_t)s * a.G + g) * 8];
                if (r[5] < r[0]) continue;
                for (int k = 0; k < 5; ++k) acc[k] += (double)(r[k + 1] - r[k]);
                t0 = r[0] < t0 ? r[0] : t0;
                t1 = r[5] > t1 ? r[5] : t1;
                ++cnt;
            }
        if (cnt)
            fprintf(stderr, "[LC_PROF] select(query) per-CTA us: setup %.2f coarse %.2f fine %.2f radix %.2f rank %.2f | span %.1f us\n",
                    acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3, acc[3] / cnt / 1e3, acc[4] / cnt / 1e3,
                    (t1 - t0) / 1e3);
    }
    return e;
}

cudaError_t launch_compact(const Arena& a, uint32_t sink, uint32_t flags, const uint32_t* buf_off,
                           const uint32_t* buf_ids, uint32_t n_slots, cudaStream_t stream) {
    CompactParams p{a, sink, flags, buf_off, buf_ids};
    const size_t smem = (size_t)a.G * bit_words(a.cap_clusters) * 4 + a.cap_clusters + 16;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    k_compact<<<n_slots, kCompactThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace lc
