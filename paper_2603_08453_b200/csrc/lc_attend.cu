// Gather-based split-K flash-decode over the selected variable-length chunks
// (north star item 3): kernels::attention (kernels.cpp:108-144) for every query
// head of a GQA group at once, over the union of the group's active spans.
//
// Data movement: each warp streams 16-token groups of gathered K/V rows into
// a private 3-stage shared-memory ring with cp.async (16-byte requests, every
// byte used; each KV row of the union is read from HBM exactly once per
// slot), so two groups are in flight while the third is computed.  The ring
// is XOR-swizzled so the fragment reads below are bank-conflict free.
//
// Math: QK^T and PV on the tensor cores (mma.sync m16n8k16, bf16 in, fp32
// accumulate) with q and the softmax weights split into bf16 hi + lo halves
// (hi in MMA rows 0..G-1, lo in rows 8..8+G-1): products carry ~16 mantissa
// bits over the exact bf16 K/V.  A per-token query mask removes (query, token)
// pairs outside that head's own active set.  Partials (m, l, o) per CTA are
// merged with log-sum-exp by the last CTA of each slot.
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

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lc {

struct AttendParams {
    Arena a;
    const float* q;  // [slot][G][D]
    float* out;      // [slot][G][D]
    unsigned long long* prof;  // optional per-CTA phase timestamps (LC_PROF=1)
};

__device__ __forceinline__ unsigned long long gtime_a() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define LC_AMARK(ph) \
    if (p.prof && threadIdx.x == 0) p.prof[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (ph)] = gtime_a();

constexpr int kAttThreads = 128;
constexpr int kAttWarps = kAttThreads / 32;
constexpr int kStages = 3;
constexpr int kWindow = 512;  // tokens expanded into shared memory at a time

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

template <int D>
__global__ void __launch_bounds__(kAttThreads, 2) k_attend(AttendParams p) {
    static_assert(D == 64 || D == 128, "D must be 64 or 128");
    constexpr int KS = D / 16;             // k-steps of QK
    constexpr int KW = D / 32;             // 16-byte chunks per thread per K row
    constexpr int NT = D / 8;              // n-tiles of PV
    constexpr int VW = D / 64;             // 16-byte chunks per thread per V row
    constexpr int ROWB = D * 2;            // bytes per K/V row
    constexpr int STAGE = 32 * ROWB;       // 16 K rows + 16 V rows
    const Arena& a = p.a;
    const uint32_t slot = a.slot0 + blockIdx.y, split = blockIdx.x, S = gridDim.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, c = lane & 3;
    const uint32_t G = a.G;

    extern __shared__ __align__(128) unsigned char dsm[];
    unsigned char* ring = dsm + (size_t)warp * kStages * STAGE;  // this warp's stages
    __shared__ uint32_t s_row[kWindow];
    __shared__ uint8_t s_msk[kWindow];
    __shared__ uint32_t s_sstart[kWindow + 1];
    __shared__ uint32_t s_slm[kWindow + 1];
    __shared__ uint32_t s_soff[kWindow + 2];
    __shared__ uint32_t s_lohi[3];
    __shared__ float s_m[kAttWarps][kMaxGroup], s_l[kAttWarps][kMaxGroup];
    __shared__ uint32_t s_last;

    LC_AMARK(0)
    const uint32_t ns = a.n_spans[slot];
    const uint32_t* soff = a.span_off + (size_t)slot * (a.cap_spans + 1);
    const Span* sp = a.spans + (size_t)slot * a.cap_spans;
    const uint32_t tot = soff[ns];
    const uint32_t beg = (uint32_t)(((unsigned long long)tot * split) / S);
    const uint32_t end = (uint32_t)(((unsigned long long)tot * (split + 1)) / S);
    const unsigned char* Kb = reinterpret_cast<const unsigned char*>(a.K + kv_off(a, slot));
    const unsigned char* Vb = reinterpret_cast<const unsigned char*>(a.V + kv_off(a, slot));
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);

    // q fragments: softmax scale and log2(e) folded in, bf16 hi (row r) + lo (row r+8)
    uint32_t qf[KS][4];
    {
        const float scale = (float)(1.4426950408889634 / sqrt((double)D));
        const float* qg = p.q + ((size_t)slot * G + (r < (int)G ? r : 0)) * D + c * (D / 4);
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            float h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) split_bf16(qg[4 * s + e] * scale, h[e], l[e]);
            const bool on = r < (int)G;
            qf[s][0] = on ? pack_bf16(h[0], h[1]) : 0u;
            qf[s][2] = on ? pack_bf16(h[2], h[3]) : 0u;
            qf[s][1] = on ? pack_bf16(l[0], l[1]) : 0u;
            qf[s][3] = on ? pack_bf16(l[2], l[3]) : 0u;
        }
    }
    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    LC_AMARK(1)

    // cp.async of one 16-token group into stage `st`: each 8-lane quarter-warp
    // copies one contiguous 128-byte half row, so every request is a full line
    auto issue = [&](uint32_t t0, uint32_t wn, int st) {
        const uint32_t sbase = ring_s + (uint32_t)st * STAGE;
        constexpr int HALVES = ROWB / 128;         // 128-byte segments per row
        constexpr int SEGS = 16 * HALVES;           // segments per 16 rows
#pragma unroll
        for (int e = 0; e < SEGS / 4; ++e) {
            const uint32_t id = 4u * e + ((uint32_t)lane >> 3);
            const uint32_t row = id / HALVES, half = id % HALVES;
            const uint32_t k = half * 8 + ((uint32_t)lane & 7);  // 16-byte chunk of the row
            const uint32_t tk = t0 + row;
            const uint32_t src_row = tk < wn ? s_row[tk] : s_row[0];
            cp_async16(sbase + row * ROWB + swz(row, k) * 16, Kb + (size_t)src_row * ROWB + k * 16);
            cp_async16(sbase + 16 * ROWB + row * ROWB + swz(row, k) * 16, Vb + (size_t)src_row * ROWB + k * 16);
        }
    };

    // first span of this split: precomputed by the span builder (k_spans) or searched
    if (tid == 0) {
        uint32_t k0 = 0;
        if (a.split_span && beg < end) {
            k0 = a.split_span[(size_t)slot * 64 + split];
        } else if (beg < end) {
            uint32_t lo = 0, hi = ns;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (soff[mid] <= beg) lo = mid;
                else hi = mid;
            }
            k0 = lo;
        }
        s_lohi[0] = k0;
        // last span of this split bounds every window's span load
        s_lohi[2] = (a.split_span && split + 1 < S) ? a.split_span[(size_t)slot * 64 + split + 1] : ns - 1;
    }
    __syncthreads();
    const uint32_t k_last = s_lohi[2];
    for (uint32_t wb = beg; wb < end; wb += kWindow) {
        const uint32_t we = min(end, wb + kWindow), wn = we - wb;
        // every span touching [wb, we) lies in [k0, k0 + wn] (spans hold >= 1 token):
        // one batched load of those spans, then all lookups in shared memory
        const uint32_t k0 = s_lohi[0];
        const uint32_t nsp = min(min(ns - k0, wn + 1), k_last + 1 - k0);
        for (uint32_t k = tid; k < nsp; k += blockDim.x) {
            const Span sk = sp[k0 + k];
            s_sstart[k] = sk.start;
            s_slm[k] = sk.len_mask;
            s_soff[k] = soff[k0 + k];
        }
        __syncthreads();
        for (uint32_t t = tid; t < kWindow; t += blockDim.x) {
            if (t < wn) {
                const uint32_t tokpos = wb + t;
                uint32_t lo = 0, hi = nsp;
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (s_soff[mid] <= tokpos) lo = mid;
                    else hi = mid;
                }
                s_row[t] = s_sstart[lo] + (tokpos - s_soff[lo]);
                s_msk[t] = (uint8_t)(s_slm[lo] & 0xffu);
                if (t == wn - 1) {  // the next window starts in the span holding token we
                    s_lohi[1] = (lo + 1 < nsp && s_soff[lo + 1] <= we) ? k0 + lo + 1 : k0 + lo;
                }
            } else {
                s_row[t] = 0;
                s_msk[t] = 0;
            }
        }
        __syncthreads();
        if (tid == 0) s_lohi[0] = s_lohi[1];

        if (wb == beg) LC_AMARK(2)
        // this warp's groups: grp = warp, warp + 4, ...
        const uint32_t ngrp = (wn + 15) / 16;
        const uint32_t my_n = ngrp > (uint32_t)warp ? (ngrp - warp + kAttWarps - 1) / kAttWarps : 0u;
#pragma unroll
        for (int st = 0; st < kStages - 1; ++st) {
            if ((uint32_t)st < my_n) issue((warp + st * kAttWarps) * 16, wn, st);
            cp_commit();
        }
        for (uint32_t it = 0; it < my_n; ++it) {
            {
                const uint32_t nxt = it + kStages - 1;
                if (nxt < my_n) issue((warp + nxt * kAttWarps) * 16, wn, (int)(nxt % kStages));
                cp_commit();
            }
            cp_wait<kStages - 1>();
            __syncwarp();
            const uint32_t t0 = (warp + it * kAttWarps) * 16;
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
            for (int w = 0; w < KW; ++w) {
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    const uint32_t row = 8 * nt + r;
                    const uint4 kv = lds128(sb + row * ROWB + swz(row, c * KW + w) * 16);
                    mma16816(sc[nt], qf[2 * w], kv.x, kv.y);
                    mma16816(sd[nt], qf[2 * w + 1], kv.z, kv.w);
                }
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) sc[nt][e] += sd[nt][e];
            // logits of query r for tokens 2c, 2c+1 (nt 0) and 8+2c, 9+2c (nt 1)
            float lg[4];
            bool ok[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int nt = x >> 1, e = x & 1;
                lg[x] = sc[nt][e] + sc[nt][2 + e];
                const uint32_t tk = nt * 8 + 2 * c + e;
                ok[x] = r < (int)G && ((s_msk[t0 + tk] >> r) & 1u);
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
            for (int w = 0; w < VW; ++w) {
                uint4 vr[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const uint32_t row = (x >> 1) * 8 + 2 * c + (x & 1);
                    vr[x] = lds128(vb + row * ROWB + swz(row, r * VW + w) * 16);
                }
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int j = w * 8 + jj, word = jj >> 1;
                    const uint32_t sel = (jj & 1) ? 0x7632u : 0x5410u;
                    auto wd = [&](const uint4& u) -> uint32_t {
                        return word == 0 ? u.x : word == 1 ? u.y : word == 2 ? u.z : u.w;
                    };
                    const uint32_t b0 = __byte_perm(wd(vr[0]), wd(vr[1]), sel);
                    const uint32_t b1 = __byte_perm(wd(vr[2]), wd(vr[3]), sel);
                    mma16816(acc[j], pa, b0, b1);
                }
            }
            __syncwarp();  // the stage is refilled by the next iteration's issue
        }
        cp_wait<0>();
        __syncthreads();
    }

    LC_AMARK(3)
    // ---- warp partial -> CTA partial (the stage ring is free now) ----
    float* s_o = reinterpret_cast<float*>(dsm);  // [warps][G][D]
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    if (r < (int)G) {
        if (c == 0) {
            s_m[warp][r] = m_run;
            s_l[warp][r] = l_run;
        }
        float* o = s_o + ((size_t)warp * G + r) * D + c * (D / 4);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            o[j] = acc[j][0] + acc[j][2];
            o[D / 8 + j] = acc[j][1] + acc[j][3];
        }
    }
    __syncthreads();
    float* part = a.partials + ((size_t)slot * S + split) * G * (D + 2);
    for (uint32_t x = tid; x < G * D; x += blockDim.x) {
        const uint32_t g = x / D, dd = x % D;
        float M = -INFINITY;
        for (int w = 0; w < kAttWarps; ++w) M = fmaxf(M, s_m[w][g]);
        float o = 0.f, L = 0.f;
        if (M != -INFINITY)
            for (int w = 0; w < kAttWarps; ++w) {
                const float f = exp2f(s_m[w][g] - M);
                o += f * s_o[((size_t)w * G + g) * D + dd];
                L += f * s_l[w][g];
            }
        part[g * (D + 2) + 2 + dd] = o;
        if (dd == 0) {
            part[g * (D + 2)] = M;
            part[g * (D + 2) + 1] = L;
        }
    }
    // ---- last CTA of the slot merges the S partials (log-sum-exp) ----
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(a.counters + slot, 1u) == S - 1 ? 1u : 0u;
    __syncthreads();
    LC_AMARK(4)
    if (!s_last) {
        LC_AMARK(5)
        return;
    }
    __threadfence();
    const float* parts = a.partials + (size_t)slot * S * G * (D + 2);
    for (uint32_t x = tid; x < G * D; x += blockDim.x) {
        const uint32_t g = x / D, dd = x % D;
        float M = -INFINITY;
        for (uint32_t s = 0; s < S; ++s) M = fmaxf(M, __ldcg(parts + (s * G + g) * (D + 2)));
        float o = 0.f, L = 0.f;
        if (M != -INFINITY)
            for (uint32_t s = 0; s < S; ++s) {
                const float* ps = parts + (s * G + g) * (D + 2);
                const float ms = __ldcg(ps);
                if (ms == -INFINITY) continue;
                const float f = exp2f(ms - M);
                o += f * __ldcg(ps + 2 + dd);
                L += f * __ldcg(ps + 1);
            }
        if (L > 0.f) {
            p.out[((size_t)slot * G + g) * D + dd] = o / L;
        } else {
            p.out[((size_t)slot * G + g) * D + dd] = 0.f;
            if (dd == 0) atomicOr(a.err, kErrEmptyActive);
        }
    }
    if (tid == 0) a.counters[slot] = 0;
    LC_AMARK(5)
}

template <int D>
static cudaError_t launch_attend_d(const AttendParams& p, dim3 grid, cudaStream_t stream) {
    // (grid.y = number of slots of this launch, starting at p.a.slot0)
    constexpr size_t ring = (size_t)kAttWarps * kStages * 32 * D * 2;
    constexpr size_t outb = (size_t)kAttWarps * kMaxGroup * D * 4;
    constexpr size_t smem = ring > outb ? ring : outb;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k_attend<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    k_attend<D><<<grid, kAttThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_attend(const Arena& a, const float* q, float* out, uint32_t n_slots, cudaStream_t stream) {
    static unsigned long long* prof = nullptr;
    const size_t nct = (size_t)a.splits * n_slots;
    if (getenv("LC_PROF") && !prof) cudaMalloc(&prof, (size_t)a.n_slots * 64 * 8 * 8);
    AttendParams p{a, q, out, prof};
    dim3 grid(a.splits, n_slots);
    cudaError_t e = a.d == 128 ? launch_attend_d<128>(p, grid, stream)
                  : a.d == 64  ? launch_attend_d<64>(p, grid, stream)
                               : cudaErrorInvalidValue;
    if (prof && e == cudaSuccess) {
        cudaStreamSynchronize(stream);
        std::vector<unsigned long long> t(nct * 8);
        cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
        double acc[5] = {0, 0, 0, 0, 0};
        unsigned long long t0 = ~0ull, t1 = 0;
        for (size_t c = 0; c < nct; ++c) {
            const unsigned long long* x = &t[c * 8];
            for (int k = 0; k < 5; ++k) acc[k] += (double)(x[k + 1] - x[k]);
            t0 = x[0] < t0 ? x[0] : t0;
            t1 = x[5] > t1 ? x[5] : t1;
        }
        fprintf(stderr, "[LC_PROF] k_attend per-CTA us: q %.2f spans %.2f stream %.2f combine %.2f merge %.2f | span %.1f us\n",
                acc[0] / nct / 1e3, acc[1] / nct / 1e3, acc[2] / nct / 1e3, acc[3] / nct / 1e3, acc[4] / nct / 1e3,
                (t1 - t0) / 1e3);
    }
    return e;
}

}  // namespace lc
