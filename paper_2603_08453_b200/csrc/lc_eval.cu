// Evaluator on the GPU: the reference's
// ground-truth oracles over a slot's live state, for audits at 128K-1M where
// the CPU versions take minutes.
//
//   audit_ub_soundness   evaluator.cpp:107-140  every query x every tier node:
//                                               max descendant chunk rep dot
//                                               <= UB + tolerance
//   oracle_topk_tokens   evaluator.cpp:43-64    the `budget` largest q.k over
//                                               the whole store, ties toward
//                                               the smaller id, sorted ids
//   full_attention       evaluator.cpp:11-41    attention over the whole store
//
// Exactness: every dot is the reference's sequential fp64 chain (float x
// float products are exact in fp64, so __fma_rn in index order reproduces
// dot_d bit for bit); qnorm * radius and the tolerance add are rounded
// separately, as the reference objects contain no FMA.  Violation counts and
// top-k id sets are therefore identical to the reference's, not approximate.
#include "../../include/lychee_b200.h"
#include "lc_common.cuh"
#include "lc_engine.hpp"

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <vector>

namespace lc {

constexpr int kAuditQ = 8;  // queries per pass (fp64 accumulators per thread)

// Upper bounds of every node for every query: one thread per (node, query
// pass), the node's centroid read in the device layout, q staged in shared
// memory as fp32.  out_f [nq][L] (internal fine ids), out_u [nq][P].
__global__ void k_audit_nodes(Arena a, uint32_t slot, const float* q, uint32_t nq, double* out_f,
                              double* out_u) {
    extern __shared__ float s_q[];  // [nq][d]
    const uint32_t d = a.d;
    const SlotState st = a.state[slot];
    for (uint32_t i = threadIdx.x; i < nq * d; i += blockDim.x) s_q[i] = q[i];
    __syncthreads();
    __shared__ double s_qn[64];
    for (uint32_t g = threadIdx.x; g < nq; g += blockDim.x) {
        double s = 0.0;  // qnorm = sqrt(sum q_j q_j), sequential (evaluator.cpp:119-121)
        for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)s_q[g * d + j], (double)s_q[g * d + j], s);
        s_qn[g] = sqrt(s);
    }
    __syncthreads();
    const uint32_t node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= st.L + st.P) return;
    const bool fine = node < st.L;
    const float* cen;
    size_t stride;  // coarse element j at cen[j * stride] (fine: row `local` of the unit's block)
    uint32_t quad_nu = 0, local = 0;
    double rad;
    if (fine) {
        const uint32_t c = node, u = a.funit[(size_t)slot * a.cap_clusters + c];
        const uint32_t base = a.unit_off[(size_t)slot * (a.cap_units + 1) + u];
        quad_nu = a.unit_off[(size_t)slot * (a.cap_units + 1) + u + 1] - base;
        local = c - base;
        cen = a.fcent + (size_t)slot * a.cap_clusters * d + (size_t)base * d;
        stride = 0;
        rad = a.frad[(size_t)slot * a.cap_clusters + c];
    } else {
        const uint32_t u = node - st.L;
        cen = a.ucent + (size_t)slot * a.cap_units * d + u;
        stride = a.cap_units;
        rad = a.urad[(size_t)slot * a.cap_units + u];
    }
    for (uint32_t g0 = 0; g0 < nq; g0 += kAuditQ) {
        double acc[kAuditQ];
#pragma unroll
        for (int k = 0; k < kAuditQ; ++k) acc[k] = 0.0;
        for (uint32_t j = 0; j < d; ++j) {
            const float c = fine ? cen[(size_t)local * d + j] : cen[(size_t)j * stride];
#pragma unroll
            for (int k = 0; k < kAuditQ; ++k)
                if (g0 + k < nq) acc[k] = __fma_rn((double)s_q[(g0 + k) * d + j], (double)c, acc[k]);
        }
#pragma unroll
        for (int k = 0; k < kAuditQ; ++k) {
            if (g0 + k >= nq) break;
            const double ub = __dadd_rn(acc[k], __dmul_rn(s_qn[g0 + k], rad));
            if (fine) out_f[(size_t)(g0 + k) * st.L + node] = ub;
            else out_u[(size_t)(g0 + k) * st.P + (node - st.L)] = ub;
        }
    }
}

// One thread per chunk: the exact dot of each query with the chunk's
// representative against its fine cluster's and coarse unit's bounds
// (evaluator.cpp:123-136: every chunk is a member of exactly one cluster,
// every cluster of exactly one unit, so this visits the reference's pairs).
__global__ void k_audit_chunks(Arena a, uint32_t slot, const float* q, uint32_t nq, const double* ub_f,
                               const double* ub_u, double tol, unsigned long long* violations) {
    extern __shared__ float s_q[];
    const uint32_t d = a.d;
    const SlotState st = a.state[slot];
    for (uint32_t i = threadIdx.x; i < nq * d; i += blockDim.x) s_q[i] = q[i];
    __syncthreads();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = 0;
    if (j < st.n_chunks) {
        const float* rep = a.chunk_rep + ((size_t)slot * a.cap_chunks + j) * d;
        const uint32_t c = a.chunk_clu[(size_t)slot * a.cap_chunks + j];
        const uint32_t u = a.funit[(size_t)slot * a.cap_clusters + c];
        for (uint32_t g0 = 0; g0 < nq; g0 += kAuditQ) {
            double acc[kAuditQ];
#pragma unroll
            for (int k = 0; k < kAuditQ; ++k) acc[k] = 0.0;
            for (uint32_t t = 0; t < d; ++t) {
                const double r = (double)rep[t];
#pragma unroll
                for (int k = 0; k < kAuditQ; ++k)
                    if (g0 + k < nq) acc[k] = __fma_rn((double)s_q[(g0 + k) * d + t], r, acc[k]);
            }
#pragma unroll
            for (int k = 0; k < kAuditQ; ++k) {
                if (g0 + k >= nq) break;
                const size_t g = g0 + k;
                if (acc[k] > __dadd_rn(ub_f[g * st.L + c], tol)) ++v;
                if (acc[k] > __dadd_rn(ub_u[g * st.P + u], tol)) ++v;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(violations, v);
}

// Exact fp64 q.k for every token of the slot, as an ascending sort key
// (descending score) plus the token id.
__global__ void k_token_scores(Arena a, uint32_t slot, const float* q, uint32_t n, unsigned long long* keys,
                               uint32_t* ids) {
    extern __shared__ float s_q[];
    const uint32_t d = a.d;
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) s_q[i] = q[i];
    __syncthreads();
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double s = 0.0;
    if (a.kv_f32) {
        const float* k = a.Kf + kv_off(a, slot) + (size_t)t * d;
        for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)s_q[j], (double)k[j], s);
    } else {
        const __nv_bfloat16* k = a.K + kv_off(a, slot) + (size_t)t * d;
        for (uint32_t j = 0; j < d; ++j) s = __fma_rn((double)s_q[j], (double)__bfloat162float(k[j]), s);
    }
    keys[t] = desc_key(s);
    ids[t] = t;
}

// rows [0, n) of a slot with every head's bit: the whole store as one active set
__global__ void k_all_rows(Arena a, uint32_t slot, uint32_t n) {
    const uint32_t all = (1u << a.G) - 1u;
    uint32_t* rows = a.rows + (size_t)slot * a.cap_tokens;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        rows[t] = t | (all << 24);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.slot_tok[slot] = n;
}

}  // namespace lc

namespace {
template <typename T>
struct DevArr {
    T* p = nullptr;
    explicit DevArr(size_t n) { lcx::ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~DevArr() { cudaFree(p); }
    DevArr(const DevArr&) = delete;
    DevArr& operator=(const DevArr&) = delete;
};
}  // namespace

extern "C" {

int lc_audit_ub(lc_index_t h, uint32_t slot, const float* queries_host, uint32_t nq, double tolerance,
                uint64_t* violations) {
    return lcx::guard([&] {
        if (!h || !queries_host || !violations || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_audit_ub: bad argument");
        sync_host(h);
        if (!h->hs[slot].loaded) lcx::fail(LC_EINVAL, "lc_audit_ub: slot not loaded");
        if (!h->a.keep_reps) lcx::fail(LC_EINVAL, "lc_audit_ub: the audit reads the chunk representatives (keep_reps = 1)");
        h->set_device();
        const Arena& a = h->a;
        const HostSlot& hs = h->hs[slot];
        *violations = 0;
        if (nq == 0) return;
        const uint32_t d = a.d;
        const size_t smem = (size_t)nq * d * 4;
        if (nq > 64 || smem > 200 * 1024) lcx::fail(LC_EINVAL, "lc_audit_ub: at most 64 queries per call");
        static KernelCfg cn, cc;
        lcx::ck(ensure_smem(k_audit_nodes, cn, smem), "smem");
        lcx::ck(ensure_smem(k_audit_chunks, cc, smem), "smem");
        DevArr<float> q((size_t)nq * d);
        DevArr<double> uf((size_t)nq * hs.L), uu((size_t)nq * hs.P);
        DevArr<unsigned long long> cnt(1);
        lcx::ck(cudaMemcpy(q.p, queries_host, (size_t)nq * d * 4, cudaMemcpyHostToDevice), "q H2D");
        lcx::ck(cudaMemset(cnt.p, 0, 8), "memset");
        const uint32_t nodes = hs.L + hs.P;
        k_audit_nodes<<<(nodes + 127) / 128, 128, smem>>>(a, slot, q.p, nq, uf.p, uu.p);
        lcx::ck(cudaGetLastError(), "k_audit_nodes");
        k_audit_chunks<<<(hs.n_chunks + 127) / 128, 128, smem>>>(a, slot, q.p, nq, uf.p, uu.p, tolerance, cnt.p);
        lcx::ck(cudaGetLastError(), "k_audit_chunks");
        unsigned long long v = 0;
        lcx::ck(cudaMemcpy(&v, cnt.p, 8, cudaMemcpyDeviceToHost), "count D2H");
        *violations = v;
    });
}

int lc_oracle_topk(lc_index_t h, uint32_t slot, const float* queries_host, uint32_t nq, uint64_t budget,
                   uint32_t* ids_out, uint64_t* n_out) {
    return lcx::guard([&] {
        if (!h || !queries_host || !ids_out || !n_out || slot >= h->a.n_slots)
            lcx::fail(LC_EINVAL, "lc_oracle_topk: bad argument");
        sync_host(h);
        if (budget < 1) lcx::fail(LC_EINVAL, "oracle_topk_tokens: budget >= 1");  // evaluator.cpp:45
        h->set_device();
        const Arena& a = h->a;
        const uint32_t n = h->hs[slot].n_tokens, d = a.d;
        const uint64_t k = std::min<uint64_t>(budget, n);
        *n_out = k;
        if (n == 0) return;
        DevArr<float> q(d);
        DevArr<unsigned long long> keys(n), keys2(n);
        DevArr<uint32_t> ids(n), ids2(n);
        size_t tmp_bytes = 0;
        lcx::ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys2.p, ids.p, ids2.p, (int)n), "cub size");
        DevArr<unsigned char> tmp(tmp_bytes);
        std::vector<uint32_t> top(k);
        for (uint32_t g = 0; g < nq; ++g) {
            lcx::ck(cudaMemcpy(q.p, queries_host + (size_t)g * d, d * 4, cudaMemcpyHostToDevice), "q H2D");
            k_token_scores<<<(n + 255) / 256, 256, d * 4>>>(a, slot, q.p, n, keys.p, ids.p);
            lcx::ck(cudaGetLastError(), "k_token_scores");
            // stable LSD radix sort: equal scores keep ascending ids (the reference's tie rule)
            lcx::ck(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys2.p, ids.p, ids2.p, (int)n), "cub sort");
            lcx::ck(cudaMemcpy(top.data(), ids2.p, k * 4, cudaMemcpyDeviceToHost), "ids D2H");
            std::sort(top.begin(), top.end());
            std::copy(top.begin(), top.end(), ids_out + (size_t)g * k);
        }
    });
}

int lc_full_attention(lc_index_t h, uint32_t slot, const float* q_dev, float* out_dev, void* stream) {
    return lcx::guard([&] {
        if (!h || !q_dev || !out_dev || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_full_attention: bad argument");
        sync_host(h);
        const uint32_t n = h->hs[slot].n_tokens;
        if (n == 0) lcx::fail(LC_EINVAL, "full_attention: empty store");  // evaluator.cpp:14
        h->set_device();
        cudaStream_t st = (cudaStream_t)stream;
        Arena a = h->a;
        k_all_rows<<<std::min<uint32_t>((n + 255) / 256, 1024), 256, 0, st>>>(a, slot, n);
        lcx::ck(cudaGetLastError(), "k_all_rows");
        a.slot0 = slot;
        // the attention kernels address q / out as [slot][G][d] arrays: shift the
        // caller's [G][d] buffers so that row `slot` lands on them
        const size_t off = (size_t)slot * a.G * a.d;
        lcx::ck(launch_attend(a, q_dev - off, out_dev - off, h->att_part, 1, st), "k_attend");
        h->last_valid = 0;  // the slot's row list no longer matches its selection
    });
}

}  // extern "C"
