// Lazy incremental update (north star item 4): KV append and the
// nearest-centroid argmax-and-graft kernel, one CTA per grafting slot.
//
// Bit-exact restatement of StreamState::flush_buffer/graft_chunk
// (streamer.cpp:29-54, 68-143) and chunk_representative (index.cpp:20-41):
// every fp64 reduction is sequential in the reference's index order, products
// that are not exact are rounded before the add (__dmul_rn/__dadd_rn), argmax
// ties keep the first candidate in the reference's scan order.
#include "lc_common.cuh"

#include <algorithm>

namespace lc {

__global__ void k_append(Arena a, const void* keys, const void* values) {
    const uint32_t slot = blockIdx.x;
    const uint32_t n = a.state[slot].n_tokens;
    if (n >= a.cap_tokens) {
        if (threadIdx.x == 0) atomicOr(a.err, kErrTokenCap);
        return;
    }
    if (a.kv_f32) {
        float* kd = a.Kf + kv_off(a, slot) + (size_t)n * a.d;
        float* vd = a.Vf + kv_off(a, slot) + (size_t)n * a.d;
        for (uint32_t j = threadIdx.x; j < a.d; j += blockDim.x) {
            kd[j] = static_cast<const float*>(keys)[(size_t)slot * a.d + j];
            vd[j] = static_cast<const float*>(values)[(size_t)slot * a.d + j];
        }
    } else {
        __nv_bfloat16* kd = a.K + kv_off(a, slot) + (size_t)n * a.d;
        __nv_bfloat16* vd = a.V + kv_off(a, slot) + (size_t)n * a.d;
        for (uint32_t j = threadIdx.x; j < a.d; j += blockDim.x) {
            kd[j] = static_cast<const __nv_bfloat16*>(keys)[(size_t)slot * a.d + j];
            vd[j] = static_cast<const __nv_bfloat16*>(values)[(size_t)slot * a.d + j];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) a.state[slot].n_tokens = n + 1;
}

struct GraftParams {
    Arena a;
    const uint32_t* take;   // [n_slots] device
    uint32_t pooling;
    void* reports;          // lc_graft_report [n_slots]
    const float* reps;      // [n_slots][d] caller-supplied representatives (graft_chunk(Chunk)), or null
    const uint32_t* kind;   // [n_slots] chunk kinds (device) or null (forced)
    const uint32_t* level;  // [n_slots] chunk levels (device) or null (0)
};

struct GraftReportDev {  // layout of lc_graft_report
    uint32_t chunk_id, cluster_id, unit_id, pad;
    double centroid_delta, fine_radius, coarse_radius;
    unsigned long long distance_comps;
};

constexpr int kGraftThreads = 256;

// block argmax over (score desc, tie key asc)
__device__ __forceinline__ void argmax_merge(double& s, uint32_t& k, double s2, uint32_t k2) {
    if (s2 > s || (s2 == s && k2 < k)) {
        s = s2;
        k = k2;
    }
}

__device__ void block_argmax(double& s, uint32_t& k, double* ws, uint32_t* wk) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const uint32_t k2 = __shfl_xor_sync(0xffffffffu, k, o);
        argmax_merge(s, k, s2, k2);
    }
    if (lane == 0) {
        ws[warp] = s;
        wk[warp] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) argmax_merge(ws[0], wk[0], ws[w], wk[w]);
    }
    __syncthreads();
    s = ws[0];
    k = wk[0];
    __syncthreads();
}

constexpr uint32_t kKeyTile = 32;     // chunk key rows staged per round
constexpr uint32_t kMemberTile = 64;  // unit member centroid rows staged per round

// n contiguous floats from global into shared memory, element x at
// dst[(x / d) * pitch + x % d]; float4 loads, up to 4 per thread in flight
__device__ __forceinline__ void stage_rows(float* dst, const float* src, uint32_t n, uint32_t d, uint32_t pitch) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    const uint32_t n4 = n / 4;
    for (uint32_t b = threadIdx.x; b < n4; b += 4 * blockDim.x) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = b + k * blockDim.x;
            if (x < n4) v[k] = __ldg(s4 + x);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = b + k * blockDim.x;
            if (x < n4) {
                const uint32_t e = 4 * x, r = e / d, j = e % d;
                float* o = dst + r * pitch + j;
                o[0] = v[k].x;
                o[1] = v[k].y;
                o[2] = v[k].z;
                o[3] = v[k].w;
            }
        }
    }
}
// n contiguous bf16 (n % 8 == 0 when d % 8 == 0) as floats into dst[x]
__device__ __forceinline__ void stage_rows_bf16(float* dst, const __nv_bfloat16* src, uint32_t n) {
    const uint4* s8 = reinterpret_cast<const uint4*>(src);
    const uint32_t n8 = n / 8;
    for (uint32_t b = threadIdx.x; b < n8; b += 2 * blockDim.x) {
        uint4 v[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t x = b + k * blockDim.x;
            if (x < n8) v[k] = __ldg(s8 + x);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t x = b + k * blockDim.x;
            if (x < n8) {
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 f = __bfloat1622float2(h[t]);
                    dst[8 * x + 2 * t] = f.x;
                    dst[8 * x + 2 * t + 1] = f.y;
                }
            }
        }
    }
}

// Sequential fp64 chains in the reference's index order, with each group of
// 8 terms loaded (and its independent products formed) before the group is
// folded in, so only the dependent add / FMA stays on the chain.  Every
// supported head dim is a multiple of 8.
__device__ __forceinline__ double seq_sumsq(const double* v, uint32_t d) {  // std::inner_product(v, v)
    double s = 0.0;
    for (uint32_t j = 0; j < d; j += 8) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = __dmul_rn(v[j + k], v[j + k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) s = __dadd_rn(s, t[k]);
    }
    return s;
}
// kernels::l2_dist (kernels.cpp:25-32): diff = (double)x - y, s += diff * diff
__device__ __forceinline__ double seq_l2(const float* x, const float* y, uint32_t ys, uint32_t d) {
    double s = 0.0;
    for (uint32_t j = 0; j < d; j += 8) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double diff = __dsub_rn((double)x[j + k], (double)y[(size_t)(j + k) * ys]);
            t[k] = __dmul_rn(diff, diff);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s = __dadd_rn(s, t[k]);
    }
    return __dsqrt_rn(s);
}
// kernels::dot (sequential FMA chain) of x with y[j * ys]
__device__ __forceinline__ double seq_dot(const float* x, const float* y, uint32_t ys, uint32_t d) {
    double s = 0.0;
    for (uint32_t j = 0; j < d; j += 8) {
        float a[8], b[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[k] = x[j + k];
            b[k] = y[(size_t)(j + k) * ys];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s = __fma_rn((double)a[k], (double)b[k], s);
    }
    return s;
}

__global__ void __launch_bounds__(kGraftThreads, 4) k_graft(GraftParams p) {
    const Arena& a = p.a;
    const uint32_t slot = blockIdx.x, tid = threadIdx.x, d = a.d;
    const uint32_t take = p.take[slot];
    if (take == 0) return;
    __shared__ double s_acc[256];
    __shared__ float s_rep[256], s_new[256], s_mu[256];
    __shared__ double s_moved[256];
    __shared__ double s_norm, s_delta, s_tonew, s_dg;
    __shared__ double ws[kGraftThreads / 32];
    __shared__ uint32_t wk[kGraftThreads / 32];
    __shared__ float s_ucol[256];  // the chosen unit's coarse centroid (dimension j)
    extern __shared__ float s_dyn[];
    SlotState* stp = a.state + slot;
    const uint32_t start = stp->chunked_end, M = stp->n_chunks, P = stp->P, L = stp->L;
    if (M >= a.cap_chunks) {
        if (tid == 0) atomicOr(a.err, kErrChunkCap);
        return;
    }
    if (take > stp->n_tokens - start) {  // the chunk must lie inside the buffered tokens
        if (tid == 0) atomicOr(a.err, kErrTake);
        return;
    }
    if (p.reps) {  // graft_chunk(Chunk): the chunk arrives with its representative
        for (uint32_t j = tid; j < d; j += blockDim.x) s_rep[j] = p.reps[(size_t)slot * d + j];
        __syncthreads();
    } else {
    // ---- chunk_representative (index.cpp:20-41) over keys [start, start+take) ----
    // the chunk's key rows stream through shared memory kKeyTile rows at a
    // time (coalesced 16-byte loads, all in flight together); thread j then
    // folds dimension j of the tile in row order, so the sequential fp64
    // chain reads shared memory instead of one dependent global load per row
    double acc = p.pooling == 0 ? 0.0 : -INFINITY;
    const size_t kbase = kv_off(a, slot) + (size_t)start * d;
    for (uint32_t i0 = 0; i0 < take; i0 += kKeyTile) {
        const uint32_t nr = min(kKeyTile, take - i0);
        if (a.kv_f32) stage_rows(s_dyn, a.Kf + kbase + (size_t)i0 * d, nr * d, d, d);
        else stage_rows_bf16(s_dyn, a.K + kbase + (size_t)i0 * d, nr * d);
        __syncthreads();
        if (tid < d) {
            if (p.pooling == 0) {
#pragma unroll 8
                for (uint32_t i = 0; i < nr; ++i) acc = __dadd_rn(acc, (double)s_dyn[i * d + tid]);
            } else {
                uint32_t i = 0;
                if (i0 == 0) acc = (double)s_dyn[tid], i = 1;
                for (; i < nr; ++i) acc = fmax(acc, (double)s_dyn[i * d + tid]);
            }
        }
        __syncthreads();
    }
    if (tid < d) s_acc[tid] = p.pooling == 0 ? __ddiv_rn(acc, (double)take) : acc;
    __syncthreads();
    if (tid == 0) {
        s_norm = __dsqrt_rn(seq_sumsq(s_acc, d));  // std::inner_product: n2 + a*a, rounded product
    }
    __syncthreads();
    if (s_norm == 0.0) {
        if (tid == 0) atomicOr(a.err, kErrZeroNorm);
        return;
    }
    for (uint32_t j = tid; j < d; j += blockDim.x) s_rep[j] = (float)__ddiv_rn(s_acc[j], s_norm);
    __syncthreads();
    }

    // ---- nearest cluster (streamer.cpp:74-106) ----
    // the slot's coarse centroids staged once, coalesced, dimension-major
    // [d][P] (dynamic shared memory): the unit scan and the coarse l2_dist read
    // them from shared memory instead of P strided global chains
    float* s_uc = s_dyn;
    const float* uc = a.ucent + (size_t)slot * a.cap_units * d;
    // (8 independent loads per thread in flight per round: the store of each
    // waits on its load, so a one-at-a-time loop paid a round trip per element)
    for (uint32_t b = tid; b < d * P; b += 8 * blockDim.x) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t x = b + k * blockDim.x;
            if (x < d * P) v[k] = __ldg(uc + (size_t)(x / P) * a.cap_units + x % P);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t x = b + k * blockDim.x;
            if (x < d * P) s_uc[x] = v[k];
        }
    }
    __syncthreads();
    const uint32_t* uoff = a.unit_off + (size_t)slot * (a.cap_units + 1);
    const float* fc = a.fcent + (size_t)slot * a.cap_clusters * d;
    const uint32_t* fo = a.forig + (size_t)slot * a.cap_clusters;
    // sequential fp64 dot (kernels::dot) of the representative with fine
    // centroid row c: the row streams in as float4 batches (4 loads in flight)
    auto row_dot = [&](uint32_t c) -> double {
        const float4* row = reinterpret_cast<const float4*>(fc + (size_t)c * d);
        double s = 0.0;
        for (uint32_t j4 = 0; j4 < d / 4; j4 += 4) {
            float4 v[4];
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) v[k] = j4 + k < d / 4 ? __ldg(row + j4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                if (j4 + k >= d / 4) break;
                const uint32_t j = 4 * (j4 + k);
                s = __fma_rn((double)s_rep[j], (double)v[k].x, s);
                s = __fma_rn((double)s_rep[j + 1], (double)v[k].y, s);
                s = __fma_rn((double)s_rep[j + 2], (double)v[k].z, s);
                s = __fma_rn((double)s_rep[j + 3], (double)v[k].w, s);
            }
        }
        return s;
    };
    unsigned long long comps = 0;
    bool scoped = !a.graft_full;
    uint32_t best_c = 0;
    if (scoped) {
        double bs = -INFINITY;
        uint32_t bu = 0xffffffffu;
        for (uint32_t u = tid; u < P; u += blockDim.x) {
            argmax_merge(bs, bu, seq_dot(s_rep, s_uc + u, P, d), u);
        }
        block_argmax(bs, bu, ws, wk);
        const uint32_t lo = uoff[bu], hi = uoff[bu + 1];
        comps = P;
        if (lo == hi) {
            scoped = false;  // empty unit: fall back to a full scan (streamer.cpp:91)
        } else {
            const uint32_t nu = hi - lo;
            double bs2 = -INFINITY;
            uint32_t bc = 0xffffffffu;
            // the unit's member rows are contiguous: stage them kMemberTile rows
            // at a time (pitch d + 1: thread t's row walk is conflict free) over
            // the coarse centroids, whose one needed column is kept in s_ucol
            for (uint32_t j = tid; j < d; j += blockDim.x) s_ucol[j] = s_uc[j * P + bu];
            __syncthreads();
            for (uint32_t t0 = 0; t0 < nu; t0 += kMemberTile) {
                const uint32_t nr = min(kMemberTile, nu - t0);
                stage_rows(s_dyn, fc + (size_t)(lo + t0) * d, nr * d, d, d + 1);
                __syncthreads();
                if (tid < nr) {
                    argmax_merge(bs2, bc, seq_dot(s_rep, s_dyn + tid * (d + 1), 1, d), lo + t0 + tid);
                }
                __syncthreads();
            }
            block_argmax(bs2, bc, ws, wk);  // stored order == internal order
            best_c = bc;
            comps += nu;
        }
    }
    if (!scoped) {
        double bs = -INFINITY;
        uint32_t bo = 0xffffffffu;
        for (uint32_t c = tid; c < L; c += blockDim.x) argmax_merge(bs, bo, row_dot(c), fo[c]);  // reference ids
        block_argmax(bs, bo, ws, wk);
        // reference id -> internal id
        for (uint32_t c = tid; c < L; c += blockDim.x)
            if (fo[c] == bo) s_acc[0] = (double)c;
        __syncthreads();
        best_c = (uint32_t)s_acc[0];
        comps = L;
        __syncthreads();
    }

    // ---- update (streamer.cpp:108-134) ----
    uint32_t* funit = a.funit + (size_t)slot * a.cap_clusters;
    uint32_t* fnmem = a.fnmem + (size_t)slot * a.cap_clusters;
    const uint32_t u = funit[best_c];
    const uint32_t lo = uoff[u], nu = uoff[u + 1] - lo, local = best_c - lo;
    float* fcw = a.fcent + (size_t)slot * a.cap_clusters * d;
    const double n = (double)fnmem[best_c];
    for (uint32_t j = tid; j < d; j += blockDim.x) {
        const float mu = fcw[fine_at(lo, nu, local, j, d)];
        s_mu[j] = mu;
        s_moved[j] = __dadd_rn(__dmul_rn(n, (double)mu), (double)s_rep[j]);
    }
    __syncthreads();
    if (tid == 0) {
        s_norm = __dsqrt_rn(seq_sumsq(s_moved, d));
    }
    __syncthreads();
    const double norm = s_norm;
    for (uint32_t j = tid; j < d; j += blockDim.x)
        s_new[j] = norm > 0.0 ? (float)__ddiv_rn(s_moved[j], norm) : s_mu[j];
    __syncthreads();
    // three sequential l2_dist (kernels.cpp:25-32) on three warps in parallel
    if (tid == 0) s_delta = seq_l2(s_new, s_mu, 1, d);
    else if (tid == 32) s_tonew = seq_l2(s_rep, s_new, 1, d);
    else if (tid == 64) {
        s_dg = scoped ? seq_l2(s_rep, s_ucol, 1, d) : seq_l2(s_rep, s_uc + u, P, d);
    }
    __syncthreads();
    __half* fcw16 = a.frow16 + (size_t)slot * a.cap_clusters * d;
    for (uint32_t j = tid; j < d; j += blockDim.x) {
        fcw[fine_at(lo, nu, local, j, d)] = s_new[j];
        fcw16[frow_at(lo, local, j, d)] = __float2half_rn(s_new[j]);
    }
    const uint32_t cid = M;
    if (a.keep_reps) {
        float* rp = a.chunk_rep + ((size_t)slot * a.cap_chunks + cid) * d;
        for (uint32_t j = tid; j < d; j += blockDim.x) rp[j] = s_rep[j];
    }
    if (tid == 0) {
        double* frad = a.frad + (size_t)slot * a.cap_clusters;
        const double r1 = __dadd_rn(frad[best_c], s_delta);
        const double rr = r1 < s_tonew ? s_tonew : r1;  // std::max(r + delta, to_new)
        frad[best_c] = rr;
        a.ftok[(size_t)slot * a.cap_clusters + best_c] += take;
        // the filters' per-row copy: radius, norm bound, token count; slot bounds raised
        double cn2 = 0.0;
        for (uint32_t j = 0; j < d; ++j) cn2 += (double)s_new[j] * (double)s_new[j];
        const float cb = norm_bound(cn2);
        const unsigned long long rb = (unsigned long long)__double_as_longlong(rr);
        a.fmeta[(size_t)slot * a.cap_clusters + best_c] =
            make_uint4((uint32_t)rb, (uint32_t)(rb >> 32), __float_as_uint(cb),
                       a.ftok[(size_t)slot * a.cap_clusters + best_c]);
        float rf = __double2float_ru(rr);
        if (rf > stp->rmax) stp->rmax = rf;
        if (cb > stp->cmax) stp->cmax = cb;
        double* ur = a.urad + (size_t)slot * a.cap_units;
        const double rg = ur[u] < s_dg ? s_dg : ur[u];  // std::max(radius, dist)
        ur[u] = rg;
        fnmem[best_c] += 1;
        uint32_t* cs = a.chunk_start + (size_t)slot * (a.cap_chunks + 1);
        cs[cid + 1] = start + take;
        a.chunk_clu[(size_t)slot * a.cap_chunks + cid] = best_c;
        a.chunk_kl[(size_t)slot * a.cap_chunks + cid] =
            (p.kind ? (p.kind[slot] & 0xffu) : 1u) | ((p.level ? p.level[slot] : 0u) << 8);
        stp->n_chunks = M + 1;
        stp->chunked_end = start + take;
        GraftReportDev* rep = reinterpret_cast<GraftReportDev*>(p.reports) + slot;
        rep->chunk_id = cid;
        rep->cluster_id = fo[best_c];
        rep->unit_id = u;
        rep->pad = 0;
        rep->centroid_delta = s_delta;
        rep->fine_radius = rr;
        rep->coarse_radius = rg;
        rep->distance_comps = comps;
    }
}

// chunk_representative (index.cpp:20-41) of rows [start, start + take) of one
// slot, for StreamState::push_token's returned Chunk: per-dim sequential fp64
// mean (or max), sequential norm, float(acc / norm).
__global__ void k_chunk_rep(Arena a, uint32_t slot, uint32_t start, uint32_t take, uint32_t pooling, float* rep) {
    __shared__ double s_acc[256];
    __shared__ double s_norm;
    const uint32_t d = a.d, tid = threadIdx.x;
    auto key = [&](uint32_t i, uint32_t j) -> double {
        return a.kv_f32 ? (double)a.Kf[kv_off(a, slot) + (size_t)(start + i) * d + j]
                        : (double)__bfloat162float(a.K[kv_off(a, slot) + (size_t)(start + i) * d + j]);
    };
    for (uint32_t j = tid; j < d; j += blockDim.x) {
        double acc;
        if (pooling == 0) {
            acc = 0.0;
            for (uint32_t i = 0; i < take; ++i) acc = __dadd_rn(acc, key(i, j));
            acc = __ddiv_rn(acc, (double)take);
        } else {
            acc = key(0, j);
            for (uint32_t i = 1; i < take; ++i) acc = fmax(acc, key(i, j));
        }
        s_acc[j] = acc;
    }
    __syncthreads();
    if (tid == 0) {
        double n2 = 0.0;
        for (uint32_t j = 0; j < d; ++j) n2 = __dadd_rn(n2, __dmul_rn(s_acc[j], s_acc[j]));
        s_norm = __dsqrt_rn(n2);
        if (s_norm == 0.0) atomicOr(a.err, kErrZeroNorm);
    }
    __syncthreads();
    for (uint32_t j = tid; j < d; j += blockDim.x) rep[j] = s_norm > 0.0 ? (float)__ddiv_rn(s_acc[j], s_norm) : 0.f;
}

// Chunk-table compaction: fold the grafted chunks [m0, M) of a slot into the
// member CSR (fmem_off / fmem), so the selection reads every member of a
// selected cluster from the CSR instead of scanning the grafted tail per head
// and step (the scan grows with the stream).  Member lists stay ascending per
// cluster (old members, then grafts in chunk order), exactly the reference's
// FineCluster::members order.  One CTA per slot; the old CSR is staged in
// shared memory first, so the rewrite is in place.  Slots with fewer than
// `min_grafted` grafted chunks are left as they are.
constexpr int kCompactThreads = 512;
__global__ void __launch_bounds__(kCompactThreads) k_compact(Arena a, uint32_t min_grafted) {
    extern __shared__ uint32_t s_c[];
    const uint32_t slot = blockIdx.x, tid = threadIdx.x;
    SlotState* stp = a.state + slot;
    const uint32_t M = stp->n_chunks, m0 = stp->m0, L = stp->L;
    if (M <= m0 || M - m0 < min_grafted) return;
    const uint32_t G = M - m0;
    uint32_t* s_wt = s_c;               // [32] scan scratch
    uint32_t* off = s_wt + 32;          // [L + 1] old offsets
    uint32_t* gpre = off + L + 1;       // [L + 1] grafted per cluster -> exclusive prefix
    uint32_t* gcl = gpre + L + 1;       // [G] cluster of each grafted chunk
    uint32_t* oldm = gcl + G;           // [off[L] = m0] old members
    uint32_t* fo = a.fmem_off + (size_t)slot * (a.cap_clusters + 1);
    uint32_t* fm = a.fmem + (size_t)slot * a.cap_chunks;
    const uint32_t* cc = a.chunk_clu + (size_t)slot * a.cap_chunks;
    for (uint32_t c = tid; c <= L; c += blockDim.x) {
        off[c] = fo[c];
        gpre[c] = 0u;
    }
    __syncthreads();
    const uint32_t nold = off[L];
    for (uint32_t k = tid; k < nold; k += blockDim.x) oldm[k] = fm[k];
    for (uint32_t j = tid; j < G; j += blockDim.x) {
        const uint32_t c = cc[m0 + j];
        gcl[j] = c;
        atomicAdd(&gpre[c], 1u);
    }
    __syncthreads();
    // exclusive prefix of the grafted counts over the clusters (block scan in tiles)
    uint32_t carry = 0;
    for (uint32_t base = 0; base <= L; base += blockDim.x) {
        const uint32_t c = base + tid;
        const uint32_t v = c <= L ? gpre[c] : 0u;
        uint32_t x = v;
        const uint32_t lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) s_wt[warp] = x;
        __syncthreads();
        uint32_t wb = 0, tot = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
            if (w < warp) wb += s_wt[w];
            tot += s_wt[w];
        }
        if (c <= L) gpre[c] = carry + wb + x - v;
        carry += tot;
        __syncthreads();
    }
    // old members shift right by the grafts of every lower cluster
    for (uint32_t k = tid; k < nold; k += blockDim.x) {
        const uint32_t m = oldm[k];
        fm[k + gpre[cc[m]]] = m;
    }
    // grafted chunk j: after its cluster's old members, in chunk order
    for (uint32_t j = tid; j < G; j += blockDim.x) {
        const uint32_t c = gcl[j];
        uint32_t rank = 0;
        for (uint32_t i = 0; i < j; ++i) rank += gcl[i] == c ? 1u : 0u;
        fm[off[c + 1] + gpre[c] + rank] = m0 + j;
    }
    for (uint32_t c = tid; c <= L; c += blockDim.x) fo[c] = off[c] + gpre[c];
    __syncthreads();
    if (tid == 0) stp->m0 = M;
}

size_t compact_smem(const Arena& a) {
    return ((size_t)2 * (a.cap_clusters + 1) + a.cap_chunks + 32) * 4;
}

cudaError_t launch_compact(const Arena& a, uint32_t min_grafted, cudaStream_t stream) {
    const size_t smem = compact_smem(a);
    static KernelCfg cfg;
    cudaError_t e = ensure_smem(k_compact, cfg, smem);
    if (e != cudaSuccess) return e;
    k_compact<<<a.n_slots, kCompactThreads, smem, stream>>>(a, min_grafted ? min_grafted : 1u);
    return cudaGetLastError();
}

cudaError_t launch_chunk_rep(const Arena& a, uint32_t slot, uint32_t start, uint32_t take, uint32_t pooling,
                             float* rep_dev, cudaStream_t stream) {
    k_chunk_rep<<<1, 256, 0, stream>>>(a, slot, start, take, pooling, rep_dev);
    return cudaGetLastError();
}

cudaError_t launch_append(const Arena& a, const void* keys, const void* values, cudaStream_t stream) {
    k_append<<<a.n_slots, 128, 0, stream>>>(a, keys, values);
    return cudaGetLastError();
}

cudaError_t launch_graft(const Arena& a, const uint32_t* take_dev, uint32_t pooling, void* reports,
                         const float* reps_dev, cudaStream_t stream, const uint32_t* kind_dev,
                         const uint32_t* level_dev) {
    GraftParams p{a, take_dev, pooling, reports, reps_dev, kind_dev, level_dev};
    // staged coarse centroids, then (aliased) unit member tiles; chunk key tiles before both
    const size_t smem = std::max<size_t>((size_t)a.d * a.cap_units * 4,
                                         std::max<size_t>((size_t)kKeyTile * a.d * 4, (size_t)kMemberTile * (a.d + 1) * 4));
    static KernelCfg cfg;
    cudaError_t e = ensure_smem(k_graft, cfg, smem);
    if (e != cudaSuccess) return e;
    k_graft<<<a.n_slots, kGraftThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace lc
