// C++ drop-in for the reference's hot path (tierkv::retrieve / retrieve_ids /
// sparse_attention and tierkv::StreamState, reference retriever.cpp and
// streamer.cpp), implemented over the C ABI (include/lychee_b200.h).
//
// The reference's callers and tests link this object in place of
// retriever.o / streamer.o; the rest of the reference
// library (types, index build, chunker, evaluator) stays as it is.  Each
// HierarchicalIndex becomes one slot of a single-head engine in the
// reference-exact mode (fp32 K/V as in TokenStore, kv_f32 = 1): selection on
// the B200 kernels (bit-exact), attention in fp64, chunk pooling and grafts on
// the device.  C ABI status codes come back as the reference's exception
// types (LC_EINVAL -> std::invalid_argument, others -> std::runtime_error).
#include "tierkv/retriever.hpp"
#include "tierkv/streamer.hpp"

#include "lychee_b200.h"
#include "tierkv/evaluator.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>

namespace tierkv {

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = lc_last_error();
    if (rc == LC_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
void ck(int rc) {
    if (rc != LC_OK) raise(rc);
}
void cuda_ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// HierarchicalIndex (index.hpp:60-73) in the C ABI's reference-numbered CSR view
struct Flat {
    std::vector<uint32_t> span, fparent, fmoff, fmem, cmoff, cmem, coc;
    std::vector<float> rep, fcent, ccent;
    std::vector<double> frad, crad;
    std::vector<uint64_t> ftok;
    lc_host_index v{};

    explicit Flat(const HierarchicalIndex& ix) {
        const size_t d = ix.dim, M = ix.chunks.size(), L = ix.fine.size(), P = ix.coarse.size();
        span.resize(M * 4);
        rep.resize(M * d);
        for (size_t j = 0; j < M; ++j) {
            const Chunk& c = ix.chunks[j];
            span[4 * j] = c.span.start;
            span[4 * j + 1] = c.span.end;
            span[4 * j + 2] = static_cast<uint32_t>(c.span.kind);
            span[4 * j + 3] = static_cast<uint32_t>(c.span.level);
            if (c.rep_key.size() == d) std::copy(c.rep_key.begin(), c.rep_key.end(), rep.begin() + j * d);
        }
        fcent.resize(L * d);
        frad.resize(L);
        ftok.resize(L);
        fparent.resize(L);
        fmoff.assign(1, 0);
        for (size_t c = 0; c < L; ++c) {
            const FineCluster& f = ix.fine[c];
            if (f.centroid.size() != d) throw std::invalid_argument("index: centroid dimension mismatch");
            std::copy(f.centroid.begin(), f.centroid.end(), fcent.begin() + c * d);
            frad[c] = f.radius;
            ftok[c] = f.token_count;
            fparent[c] = f.parent_unit;
            fmem.insert(fmem.end(), f.members.begin(), f.members.end());
            fmoff.push_back(static_cast<uint32_t>(fmem.size()));
        }
        ccent.resize(P * d);
        crad.resize(P);
        cmoff.assign(1, 0);
        for (size_t u = 0; u < P; ++u) {
            const CoarseUnit& cu = ix.coarse[u];
            if (cu.centroid.size() != d) throw std::invalid_argument("index: centroid dimension mismatch");
            std::copy(cu.centroid.begin(), cu.centroid.end(), ccent.begin() + u * d);
            crad[u] = cu.radius;
            cmem.insert(cmem.end(), cu.members.begin(), cu.members.end());
            cmoff.push_back(static_cast<uint32_t>(cmem.size()));
        }
        coc = ix.cluster_of_chunk;
        v.dim = static_cast<uint32_t>(d);
        v.n_chunks = static_cast<uint32_t>(M);
        v.n_clusters = static_cast<uint32_t>(L);
        v.n_units = static_cast<uint32_t>(P);
        v.chunk_span = span.data();
        v.chunk_rep = rep.data();
        v.fine_centroid = fcent.data();
        v.fine_radius = frad.data();
        v.fine_token_count = ftok.data();
        v.fine_parent = fparent.data();
        v.fine_member_off = fmoff.data();
        v.fine_members = fmem.data();
        v.coarse_centroid = ccent.data();
        v.coarse_radius = crad.data();
        v.coarse_member_off = cmoff.data();
        v.coarse_members = cmem.data();
        v.cluster_of_chunk = coc.data();
    }
};

// one single-head slot on the GPU and its small device-side staging buffers
struct Engine {
    lc_index_t h = nullptr;
    uint32_t d = 0, cap_tokens = 0;
    float* q_dev = nullptr;
    float* out_dev = nullptr;
    float* kv_dev = nullptr;  // [2][d] one appended token
    uint32_t* boff_dev = nullptr;
    uint32_t* bids_dev = nullptr;
    size_t bids_cap = 0;
    lc_graft_report* rep_dev = nullptr;
    // the engine's own stream and page-locked staging: a call's copies and
    // kernels are queued asynchronously and the host waits once
    cudaStream_t st = nullptr;
    float* h_io = nullptr;     // [2][d]: q in, output out
    uint32_t* h_ids = nullptr; // [2 + bids_cap]: buffer offsets then ids

    Engine(uint32_t dim, uint32_t cap_tokens_, uint32_t cap_chunks, uint32_t cap_clusters, uint32_t cap_units,
           bool graft_full, uint32_t pooling)
        : d(dim), cap_tokens(cap_tokens_) {
        lc_index_desc desc{};
        desc.n_slots = 1;
        desc.dim = dim;
        desc.group = 1;
        desc.cap_tokens = std::max<uint32_t>(cap_tokens_, 1);
        desc.cap_chunks = std::max<uint32_t>(cap_chunks, 1);
        desc.cap_clusters = std::max<uint32_t>(cap_clusters, 1);
        desc.cap_units = std::max<uint32_t>(cap_units, 1);
        desc.structure_aware = 1;
        desc.graft_full = graft_full ? 1 : 0;
        desc.keep_reps = 1;
        desc.pooling = pooling;
        desc.kv_f32 = 1;
        int dev = 0;
        cuda_ck(cudaGetDevice(&dev), "cudaGetDevice");
        desc.device = dev;
        ck(lc_index_create(&desc, &h));
        cuda_ck(cudaMalloc(&q_dev, d * 4), "cudaMalloc q");
        cuda_ck(cudaMalloc(&out_dev, d * 4), "cudaMalloc out");
        cuda_ck(cudaMalloc(&kv_dev, 2 * d * 4), "cudaMalloc kv");
        cuda_ck(cudaMalloc(&boff_dev, 2 * 4), "cudaMalloc buffer offsets");
        cuda_ck(cudaMalloc(&rep_dev, sizeof(lc_graft_report)), "cudaMalloc report");
        // a blocking stream: ordered with the legacy-stream calls of the ABI
        // (k_append, k_chunk_rep, downloads) without extra events
        cuda_ck(cudaStreamCreateWithFlags(&st, cudaStreamDefault), "stream");
        cuda_ck(cudaMallocHost(&h_io, 2 * d * 4), "cudaMallocHost io");
    }
    ~Engine() {
        if (h) lc_index_destroy(h);
        cudaFree(q_dev);
        cudaFree(out_dev);
        cudaFree(kv_dev);
        cudaFree(boff_dev);
        cudaFree(bids_dev);
        cudaFree(rep_dev);
        if (st) cudaStreamDestroy(st);
        cudaFreeHost(h_io);
        cudaFreeHost(h_ids);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void upload(const HierarchicalIndex& ix, const TokenStore& store) {
        const Flat f(ix);
        const uint32_t n = static_cast<uint32_t>(store.size());
        if (ix.chunks.empty()) {  // degenerate-only index: the store alone
            ck(lc_kv_upload_slot(h, 0, store.keys_flat().data(), store.values_flat().data(), n));
            return;
        }
        ck(lc_index_upload_slot(h, 0, &f.v, store.keys_flat().data(), store.values_flat().data(), n));
    }

    void buffer_list(std::span<const uint32_t> ids) {
        if (ids.size() > bids_cap || !bids_dev) {
            cuda_ck(cudaStreamSynchronize(st), "sync");
            cudaFree(bids_dev);
            cudaFreeHost(h_ids);
            bids_dev = nullptr;
            h_ids = nullptr;
            bids_cap = std::max<size_t>(ids.size(), 64);
            cuda_ck(cudaMalloc(&bids_dev, bids_cap * 4), "cudaMalloc buffer ids");
            cuda_ck(cudaMallocHost(&h_ids, (bids_cap + 2) * 4), "cudaMallocHost buffer ids");
        }
        h_ids[0] = 0;
        h_ids[1] = static_cast<uint32_t>(ids.size());
        std::copy(ids.begin(), ids.end(), h_ids + 2);
        cuda_ck(cudaMemcpyAsync(boff_dev, h_ids, 8, cudaMemcpyHostToDevice, st), "buffer offsets");
        if (!ids.empty())
            cuda_ck(cudaMemcpyAsync(bids_dev, h_ids + 2, ids.size() * 4, cudaMemcpyHostToDevice, st), "buffer ids");
    }

    // sticky device conditions of the last calls, as the reference's exceptions
    void device_errors() {
        uint32_t bits = 0;
        ck(lc_device_error(h, &bits, 1));
        if (!bits) return;
        if (bits & (1u << 6)) throw std::invalid_argument("sparse_attention: empty active set");
        if (bits & (1u << 1)) throw std::invalid_argument("select_topk: k must be >= 1");
        throw std::runtime_error("device error bits " + std::to_string(bits));
    }
};

// 64-bit word hash (8 bytes per step; the tail byte-wise)
uint64_t mix(uint64_t h, const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = (h ^ w) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
    }
    for (; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
template <typename T>
uint64_t mixv(uint64_t h, const T& x) {
    return mix(h, &x, sizeof x);
}

// The engine cache key of a (HierarchicalIndex, TokenStore) pair: identity
// (addresses, sizes, the node arrays' buffers) plus a digest of every
// cluster's and unit's radius, token count, parent and member count, one
// coordinate of every 8th fine centroid, a strided sample of the coarse centroids,
// chunk spans and chunk -> cluster map, and a sample of the store's rows
// (~30 K words at 128K, ~0.1 ms; the round-1 key hashed every centroid
// byte-wise on every call, ~2.5 ms).  An in-place edit of a field outside
// the digest on the same index object between calls is not seen; build a new
// index or touch a digested field (e.g. a radius) after such an edit.
uint64_t store_key(uint64_t h, const TokenStore& s) {
    const size_t n = s.size(), d = s.dim();
    h = mixv(h, &s);
    h = mixv(h, n);
    h = mixv(h, d);
    for (const auto arr : {s.keys_flat(), s.values_flat()}) {
        h = mixv(h, arr.data());
        const size_t step = std::max<size_t>(1, arr.size() / 1024);
        for (size_t i = 0; i < arr.size(); i += step) h = mixv(h, arr[i]);
        if (!arr.empty()) h = mix(h, arr.data() + (arr.size() - std::min<size_t>(arr.size(), d)),
                                  std::min<size_t>(arr.size(), d) * 4);
    }
    return h;
}

uint64_t fingerprint(const HierarchicalIndex& ix) {
    uint64_t h = 1469598103934665603ull;
    const size_t d = ix.dim;
    h = mixv(h, &ix);
    h = mixv(h, d);
    h = mixv(h, ix.chunks.size());
    h = mixv(h, ix.fine.size());
    h = mixv(h, ix.coarse.size());
    h = mixv(h, ix.chunks.data());
    h = mixv(h, ix.fine.data());
    h = mixv(h, ix.coarse.data());
    // chunk spans and chunk -> cluster: a fixed stride (they only change by
    // appending, which changes the sizes above)
    for (size_t c = 0; c < ix.chunks.size(); c += 16) h = mixv(h, ix.chunks[c].span.start);
    if (!ix.chunks.empty()) h = mixv(h, ix.chunks.back().span.end);
    for (size_t c = 0; c < ix.cluster_of_chunk.size(); c += 16) h = mixv(h, ix.cluster_of_chunk[c]);
    // every cluster's scalar fields and member count (contiguous structs), and
    // one centroid coordinate of every 8th cluster (each is a pointer chase
    // into its own allocation; the fp64 radii already pin every cluster)
    for (size_t c = 0; c < ix.fine.size(); ++c) {
        const FineCluster& f = ix.fine[c];
        h = mixv(h, f.radius);
        h = mixv(h, (uint64_t)f.token_count ^ ((uint64_t)f.parent_unit << 40) ^ ((uint64_t)f.members.size() << 52));
        if ((c & 7) == 0 && !f.centroid.empty()) h = mixv(h, f.centroid[f.centroid.size() / 2]);
    }
    for (const CoarseUnit& u : ix.coarse) {
        h = mixv(h, u.radius);
        h = mixv(h, u.members.size());
        for (size_t j = 0; j < u.centroid.size(); j += 16) h = mixv(h, u.centroid[j]);
    }
    return ix.store ? store_key(h, *ix.store) : h;
}

uint64_t fingerprint(const TokenStore& s) { return store_key(1469598103934665603ull, s); }

// a few engines kept per thread, keyed by content
struct CacheEntry {
    uint64_t key = 0;
    std::unique_ptr<Engine> e;
};
thread_local std::vector<CacheEntry> g_cache;

Engine& cached(uint64_t key, const std::function<std::unique_ptr<Engine>()>& make) {
    for (auto& c : g_cache)
        if (c.key == key && c.e) return *c.e;
    if (g_cache.size() >= 4) g_cache.erase(g_cache.begin());
    g_cache.push_back({key, make()});
    return *g_cache.back().e;
}

lc_budgets to_c(const Budgets& b) {
    lc_budgets c{};
    c.unit_topk = b.unit_topk;
    c.mode = b.mode == SelectionMode::token_budget ? LC_MODE_TOKEN_BUDGET : LC_MODE_FIXED_CLUSTER_COUNT;
    c.cluster_topk = b.cluster_topk;
    c.token_budget = b.token_budget;
    c.sink_size = b.sink_size;
    return c;
}

// retrieve_ids / retrieve (retriever.cpp:78-167) for one query on a slot
// whose device state mirrors `ix` / `store`
RetrievalResult run_retrieve(Engine& e, const HierarchicalIndex& ix, const TokenStore& store,
                             std::span<const float> q, const Budgets& budgets, std::span<const uint32_t> buffer_ids,
                             bool attend) {
    budgets.validate();
    if (q.size() != store.dim()) throw std::invalid_argument("retrieve: query dimension mismatch");
    const size_t n = store.size();
    std::vector<uint32_t> buf(buffer_ids.begin(), buffer_ids.end());  // collect_active sorts and dedups
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
    if (!buf.empty() && buf.back() >= n) throw std::invalid_argument("retrieve: buffer id outside the store");
    RetrievalResult res;
    const bool fits = budgets.mode == SelectionMode::token_budget && n <= budgets.token_budget;
    if (ix.chunks.empty() && !fits) {
        // no chunks: the reference degenerates to every token (retriever.cpp:89)
        res.degenerate = true;
        res.selected_units.resize(ix.coarse.size());
        std::iota(res.selected_units.begin(), res.selected_units.end(), 0u);
        res.selected_clusters.resize(ix.fine.size());
        std::iota(res.selected_clusters.begin(), res.selected_clusters.end(), 0u);
        res.active_token_ids.resize(n);
        std::iota(res.active_token_ids.begin(), res.active_token_ids.end(), 0u);
        if (attend) res.output = sparse_attention(q, store, res.active_token_ids);
        return res;
    }
    static const bool prof = getenv("TIERKV_DROPIN_PROF") != nullptr;  // diagnostics: per-phase host times
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    std::copy(q.begin(), q.end(), e.h_io);
    cuda_ck(cudaMemcpyAsync(e.q_dev, e.h_io, q.size() * 4, cudaMemcpyHostToDevice, e.st), "q H2D");
    e.buffer_list(buf);
    const lc_budgets b = to_c(budgets);
    const auto t1 = now();
    ck(lc_retrieve(e.h, e.q_dev, &b, LC_BUFFER_LIST, e.boff_dev, e.bids_dev, attend ? e.out_dev : nullptr, e.st));
    if (attend)
        cuda_ck(cudaMemcpyAsync(e.h_io + e.d, e.out_dev, store.dim() * 4, cudaMemcpyDeviceToHost, e.st), "out D2H");
    // the selection rides the same stream into page-locked staging: one wait per call
    ck(lc_selection_stage(e.h, 0, 0, e.st));
    const auto t2 = now();
    cuda_ck(cudaStreamSynchronize(e.st), "retrieve");
    const auto t3 = now();
    lc_selection_info info{};
    ck(lc_selection_read_staged(e.h, &info, nullptr, 0, nullptr, 0, nullptr, 0));  // sizes first
    // (no zero-filled n-token vectors per call: exact sizes, then the copies)
    res.selected_units.resize(info.degenerate ? ix.coarse.size() : info.n_units);
    res.selected_clusters.resize(info.degenerate ? ix.fine.size() : info.n_clusters);
    res.active_token_ids.resize(info.n_active);
    ck(lc_selection_read_staged(e.h, &info, res.selected_units.data(), res.selected_units.size(),
                                res.selected_clusters.data(), res.selected_clusters.size(),
                                res.active_token_ids.data(), res.active_token_ids.size()));
    if (prof) {
        const auto t4 = now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "[dropin] stage %.1f launch %.1f device %.1f download %.1f us\n", us(t0, t1), us(t1, t2),
                     us(t2, t3), us(t3, t4));
    }
    if (info.error) e.device_errors();  // sticky bits: raise the reference's exception and clear them
    res.selected_units.resize(info.n_units);
    res.selected_clusters.resize(info.n_clusters);
    res.active_token_ids.resize(info.n_active);
    res.scanned_centroids = info.scanned_centroids;
    res.degenerate = info.degenerate != 0;
    if (attend) res.output.assign(e.h_io + e.d, e.h_io + e.d + store.dim());
    return res;
}

RetrievalResult retrieve_impl(const HierarchicalIndex& index, std::span<const float> q, const Budgets& budgets,
                              std::span<const uint32_t> buffer_ids, bool attend) {
    budgets.validate();
    if (!index.store) throw std::invalid_argument("retrieve: index has no token store");
    const TokenStore& store = *index.store;
    if (q.size() != store.dim()) throw std::invalid_argument("retrieve: query dimension mismatch");
    const uint64_t key = fingerprint(index);
    Engine& e = cached(key, [&] {
        auto e = std::make_unique<Engine>(static_cast<uint32_t>(index.dim), static_cast<uint32_t>(store.size()),
                                          static_cast<uint32_t>(index.chunks.size()),
                                          static_cast<uint32_t>(index.fine.size()),
                                          static_cast<uint32_t>(index.coarse.size()), false,
                                          index.config.pooling == Pooling::max ? 1u : 0u);
        e->upload(index, store);
        return e;
    });
    return run_retrieve(e, index, store, q, budgets, buffer_ids, attend);
}

}  // namespace

void Budgets::validate() const {  // retriever.cpp:11-17
    if (unit_topk < 1) throw std::invalid_argument("unit_topk must be >= 1");
    if (mode == SelectionMode::fixed_cluster_count && cluster_topk < 1)
        throw std::invalid_argument("cluster_topk must be >= 1");
    if (mode == SelectionMode::token_budget && token_budget < 1)
        throw std::invalid_argument("token_budget must be >= 1");
}

// retriever.cpp:19-25: sequential fp64 dot + ||q|| r (kernels::dot / l2_norm)
double score_upper_bound(std::span<const float> q, std::span<const float> centroid, double radius) {
    if (q.size() != centroid.size()) throw std::invalid_argument("score_upper_bound: dimension mismatch");
    double dot = 0.0, n2 = 0.0;
    for (size_t j = 0; j < q.size(); ++j) {
        dot += static_cast<double>(q[j]) * static_cast<double>(centroid[j]);
        n2 += static_cast<double>(q[j]) * static_cast<double>(q[j]);
    }
    return dot + std::sqrt(n2) * radius;
}

// retriever.cpp:27-39: (score desc, id asc), truncated to k
std::vector<uint32_t> select_topk(std::span<const std::pair<uint32_t, double>> scores, size_t k) {
    if (k < 1) throw std::invalid_argument("select_topk: k must be >= 1");
    std::vector<std::pair<uint32_t, double>> s(scores.begin(), scores.end());
    std::stable_sort(s.begin(), s.end(), [](const auto& a, const auto& b) {
        return a.second != b.second ? a.second > b.second : a.first < b.first;
    });
    s.resize(std::min(k, s.size()));
    std::vector<uint32_t> ids(s.size());
    for (size_t i = 0; i < s.size(); ++i) ids[i] = s[i].first;
    return ids;
}

RetrievalResult retrieve_ids(const HierarchicalIndex& index, std::span<const float> q, const Budgets& budgets,
                             std::span<const uint32_t> buffer_ids) {
    return retrieve_impl(index, q, budgets, buffer_ids, false);
}

RetrievalResult retrieve(const HierarchicalIndex& index, std::span<const float> q, const Budgets& budgets,
                         std::span<const uint32_t> buffer_ids) {
    return retrieve_impl(index, q, budgets, buffer_ids, true);
}

// retriever.cpp:41-50 on the device (fp64 softmax over the given rows)
VecF sparse_attention(std::span<const float> q, const TokenStore& store, std::span<const uint32_t> ids) {
    if (ids.empty()) throw std::invalid_argument("sparse_attention: empty active set");
    if (q.size() != store.dim()) throw std::invalid_argument("sparse_attention: query dimension mismatch");
    Engine& e = cached(fingerprint(store) ^ 0x5bd1e995ull, [&] {
        auto e = std::make_unique<Engine>(static_cast<uint32_t>(store.dim()), static_cast<uint32_t>(store.size()), 1,
                                          1, 1, false, 0);
        ck(lc_kv_upload_slot(e->h, 0, store.keys_flat().data(), store.values_flat().data(),
                             static_cast<uint32_t>(store.size())));
        return e;
    });
    cuda_ck(cudaMemcpy(e.q_dev, q.data(), q.size() * 4, cudaMemcpyHostToDevice), "q H2D");
    ck(lc_sparse_attention_ids(e.h, 0, e.q_dev, ids.data(), static_cast<uint32_t>(ids.size()), e.out_dev, nullptr));
    e.device_errors();
    VecF out(store.dim());
    cuda_ck(cudaMemcpy(out.data(), e.out_dev, out.size() * 4, cudaMemcpyDeviceToHost), "out D2H");
    return out;
}

// ---------------------------------------------------------------------------
// StreamState (streamer.cpp:13-165)

struct StreamDevice {
    Engine e;
    size_t dev_end = 0;  // end of the last chunk the device holds
    uint32_t cap_chunks = 0;
    StreamDevice(uint32_t d, uint32_t cap_tokens, uint32_t cap_chunks_, uint32_t L, uint32_t P, bool full, uint32_t pool)
        : e(d, cap_tokens, cap_chunks_, L, P, full, pool), cap_chunks(cap_chunks_) {}
};

namespace {
constexpr uint32_t kStreamGrowth = 1u << 14;  // initial decode-time token / chunk headroom of a stream engine

// a fresh engine for the stream's current host mirrors, with room for `extra`
// more tokens and chunks (the engine is re-created when a stream outgrows it)
std::unique_ptr<StreamDevice> open_stream(const HierarchicalIndex& ix, const TokenStore& store,
                                          const StreamerConfig& cfg, uint32_t extra) {
    auto dev = std::make_unique<StreamDevice>(
        static_cast<uint32_t>(ix.dim), static_cast<uint32_t>(store.size()) + extra,
        static_cast<uint32_t>(ix.chunks.size()) + extra, static_cast<uint32_t>(ix.fine.size()),
        static_cast<uint32_t>(ix.coarse.size()), cfg.graft_search == GraftSearch::full,
        ix.config.pooling == Pooling::max ? 1u : 0u);
    dev->e.upload(ix, store);
    dev->dev_end = ix.chunks.empty() ? 0 : ix.chunks.back().span.end;
    return dev;
}

}  // namespace

StreamState::StreamState(TokenStore store, HierarchicalIndex index, StreamerConfig cfg)
    : store_(std::move(store)), index_(std::move(index)), cfg_(std::move(cfg)) {
    cfg_.policy.validate();
    if (index_.fine.empty()) throw std::invalid_argument("stream state: empty index");
    index_.store = &store_;
    chunked_end_ = index_.chunks.empty() ? 0 : index_.chunks.back().span.end;
    if (chunked_end_ > store_.size()) throw std::invalid_argument("stream state: chunks exceed store");
    dev_ = open_stream(index_, store_, cfg_, kStreamGrowth);
}

StreamState::~StreamState() = default;

std::vector<uint32_t> StreamState::buffer_ids() const {
    std::vector<uint32_t> ids(store_.size() - chunked_end_);
    std::iota(ids.begin(), ids.end(), static_cast<uint32_t>(chunked_end_));
    return ids;
}

// streamer.cpp:29-54: the host chunker picks the chunk, the device pools it
std::optional<Chunk> StreamState::flush_buffer() {
    const size_t len = buffer_size();
    const ChunkPolicy& pol = cfg_.policy;
    size_t take = pol.max_len;
    BoundaryKind kind = BoundaryKind::forced;
    int level = 0;
    if (cfg_.structure_aware) {
        std::vector<std::string> texts(len);
        for (size_t i = 0; i < len; ++i) texts[i] = store_.text(chunked_end_ + i);
        auto spans = segment(texts, pol);
        const ChunkSpan& head = spans.front();
        if (head.kind != BoundaryKind::tail) {
            take = head.length();
            kind = head.kind;
            level = head.level;
        }
    }
    Chunk chunk;
    chunk.span = {static_cast<uint32_t>(chunked_end_), static_cast<uint32_t>(chunked_end_ + take), kind, level};
    chunk.rep_key.resize(store_.dim());
    ck(lc_chunk_rep(dev_->e.h, 0, static_cast<uint32_t>(chunked_end_), static_cast<uint32_t>(take),
                    chunk.rep_key.data()));
    chunked_end_ += take;
    return chunk;
}

std::optional<Chunk> StreamState::push_token(const TokenRecord& token) {
    store_.append(token);  // rejects non-sequential ids and dimension mismatches
    if (store_.size() > dev_->e.cap_tokens || index_.chunks.size() + 1 >= dev_->cap_chunks) {
        // outgrown: a larger engine from the host mirrors (the new token included)
        const size_t dev_end = dev_->dev_end;
        dev_ = open_stream(index_, store_, cfg_, std::max<uint32_t>(kStreamGrowth, (uint32_t)store_.size()));
        dev_->dev_end = dev_end;
    } else {
        const size_t d = store_.dim();
        cuda_ck(cudaMemcpy(dev_->e.kv_dev, token.key.data(), d * 4, cudaMemcpyHostToDevice), "key H2D");
        cuda_ck(cudaMemcpy(dev_->e.kv_dev + d, token.value.data(), d * 4, cudaMemcpyHostToDevice), "value H2D");
        ck(lc_kv_append(dev_->e.h, dev_->e.kv_dev, dev_->e.kv_dev + d, nullptr));
    }
    std::optional<Chunk> emitted;
    if (buffer_size() >= cfg_.policy.max_len) emitted = flush_buffer();
    while (buffer_size() >= cfg_.max_buffer) {  // the reference's hard cap (unreachable under the eager flush)
        auto extra = flush_buffer();
        if (extra) graft_chunk(std::move(*extra));
    }
    return emitted;
}

// streamer.cpp:68-143 on the device; the host mirror is refreshed from it
GraftReport StreamState::graft_chunk(Chunk chunk) {
    if (index_.fine.empty()) throw std::invalid_argument("graft: empty index");
    if (chunk.rep_key.size() != index_.dim) throw std::invalid_argument("graft: representative dimension mismatch");
    if (chunk.span.start != dev_->dev_end || chunk.span.end <= chunk.span.start)
        throw std::invalid_argument("graft: the chunk must directly follow the indexed chunks");
    const uint32_t take = chunk.span.length(), kind = static_cast<uint32_t>(chunk.span.kind),
                   level = static_cast<uint32_t>(chunk.span.level);
    ck(lc_graft_rep(dev_->e.h, &take, &kind, &level, chunk.rep_key.data(), dev_->e.rep_dev, nullptr));
    dev_->e.device_errors();
    lc_graft_report r{};
    cuda_ck(cudaMemcpy(&r, dev_->e.rep_dev, sizeof r, cudaMemcpyDeviceToHost), "report D2H");
    dev_->dev_end += take;
    ++graft_count_;
    // patch the host mirror the way the reference's graft mutates its index
    // (streamer.cpp:108-134): one cluster (centroid, radius, token count,
    // members), one unit (radius), one appended chunk
    if (r.cluster_id >= index_.fine.size() || r.unit_id >= index_.coarse.size() || r.chunk_id != index_.chunks.size())
        throw std::runtime_error("graft: device report does not match the host index");
    FineCluster& fc = index_.fine[r.cluster_id];
    uint64_t tok = 0;
    ck(lc_cluster_download(dev_->e.h, 0, r.cluster_id, fc.centroid.data(), &fc.radius, &tok));
    fc.token_count = static_cast<size_t>(tok);
    fc.members.push_back(r.chunk_id);
    index_.coarse[r.unit_id].radius = r.coarse_radius;
    index_.cluster_of_chunk.push_back(r.cluster_id);
    index_.chunks.push_back(std::move(chunk));
    GraftReport report;
    report.chunk_id = r.chunk_id;
    report.cluster_id = r.cluster_id;
    report.unit_id = r.unit_id;
    report.centroid_delta = r.centroid_delta;
    report.fine_radius = r.fine_radius;
    report.coarse_radius = r.coarse_radius;
    report.distance_comps = r.distance_comps;
    return report;
}

// streamer.cpp:145-165
DecodeOutcome StreamState::decode_step(std::span<const float> q, const TokenRecord& token, const Budgets& budgets) {
    DecodeOutcome out;
    auto buffered = buffer_ids();
    out.retrieval = run_retrieve(dev_->e, index_, store_, q, budgets, buffered, true);
    std::vector<uint32_t> selected = out.retrieval.selected_clusters;
    std::sort(selected.begin(), selected.end());
    static const std::vector<uint32_t> empty_set;
    out.jaccard = eval::jaccard(history_.empty() ? empty_set : history_.back(), selected);
    std::vector<std::vector<uint32_t>> window(history_.begin(), history_.end());
    out.window_hit = eval::window_hit(window, selected);
    history_.push_back(std::move(selected));
    while (history_.size() > cfg_.history_capacity) history_.pop_front();
    if (auto chunk = push_token(token)) out.graft = graft_chunk(std::move(*chunk));
    return out;
}

}  // namespace tierkv
