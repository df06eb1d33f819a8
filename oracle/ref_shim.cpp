// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim around the UNMODIFIED reference library (tierkv, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It exists
// so that tests/ (and bench.py's cpu_baseline / --impl reference legs) can
// drive the reference through ctypes: generate the reference's synthetic
// workloads, build its HierarchicalIndex, run retrieve()/decode_step(), export
// every field of the index and time the reference path on the host cores.
//
// Nothing in the product (paper_2603_08453_b200/) links or calls this file.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for any other std::exception (error text via tkr_last_error()).

#include "tierkv/chunker.hpp"
#include "tierkv/evaluator.hpp"
#include "tierkv/index.hpp"
#include "tierkv/kernels.hpp"
#include "tierkv/retriever.hpp"
#include "tierkv/serialize.hpp"
#include "tierkv/streamer.hpp"
#include "tierkv/workload.hpp"

#include <chrono>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace tierkv;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct WorkloadH {
    WorkloadSpec spec;
    Workload w;
};

// A StreamState owns the store and index; standalone retrieve() calls read
// state.index() exactly as the reference bench does (bench.cpp:104).
struct EngineH {
    std::unique_ptr<StreamState> state;
};

Budgets make_budgets(uint32_t unit_topk, uint32_t mode, uint32_t cluster_topk,
                     uint64_t token_budget, uint32_t sink) {
    Budgets b;
    b.unit_topk = unit_topk;
    b.mode = mode == 0 ? SelectionMode::fixed_cluster_count : SelectionMode::token_budget;
    b.cluster_topk = cluster_topk;
    b.token_budget = token_budget;
    b.sink_size = sink;
    return b;
}

TokenStore make_store(const float* keys, const float* values, const uint8_t* text_code,
                      uint64_t n, uint64_t d) {
    TokenStore store(d);
    for (uint64_t i = 0; i < n; ++i) {
        TokenRecord t;
        t.id = static_cast<uint32_t>(i);
        t.text = text_code ? std::string(text_code[i] == 1 ? "\n" : text_code[i] == 2 ? "}" : "")
                           : std::string();
        t.key.assign(keys + i * d, keys + (i + 1) * d);
        t.value.assign(values + i * d, values + (i + 1) * d);
        store.append(t);
    }
    return store;
}

void copy_ids(const std::vector<uint32_t>& v, uint32_t* out, uint64_t cap) {
    if (!out) return;
    std::memcpy(out, v.data(), sizeof(uint32_t) * std::min<uint64_t>(cap, v.size()));
}

void write_result(const RetrievalResult& r, uint32_t* units, uint64_t units_cap,
                  uint32_t* clusters, uint64_t clusters_cap, uint32_t* active,
                  uint64_t active_cap, float* output, uint64_t* counts) {
    copy_ids(r.selected_units, units, units_cap);
    copy_ids(r.selected_clusters, clusters, clusters_cap);
    copy_ids(r.active_token_ids, active, active_cap);
    if (output && !r.output.empty())
        std::memcpy(output, r.output.data(), sizeof(float) * r.output.size());
    if (counts) {
        counts[0] = r.selected_units.size();
        counts[1] = r.selected_clusters.size();
        counts[2] = r.active_token_ids.size();
        counts[3] = r.scanned_centroids;
        counts[4] = r.degenerate ? 1 : 0;
    }
}

}  // namespace

extern "C" {

const char* tkr_last_error() { return g_err.c_str(); }

int tkr_threads() { return kernels::thread_count(); }

// OpenMP team size for parallel regions started by the calling host thread
// (bench's threaded CPU baseline runs one single-threaded engine per thread)
void tkr_set_thread_team(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}

// ---- workload (workload.cpp:110-169) -------------------------------------
int tkr_workload_new(uint64_t n_tokens, uint64_t d, uint64_t n_blobs, double concentration,
                     uint64_t query_count, double locality, uint64_t seed, void** out) {
    return guard([&] {
        auto h = std::make_unique<WorkloadH>();
        h->spec.n_tokens = n_tokens;
        h->spec.d = d;
        h->spec.n_blobs = n_blobs;
        h->spec.blob_concentration = concentration;
        h->spec.query_count = query_count;
        h->spec.query_locality = locality;
        h->spec.seed = seed;
        h->w = gen_clustered_workload(h->spec);
        *out = h.release();
    });
}

void tkr_workload_free(void* h) { delete static_cast<WorkloadH*>(h); }

// keys/values [n*d], text codes [n] (0 "", 1 "\n", 2 other), queries [qc*d],
// centers [n_blobs*d], token_blob [n]
void tkr_workload_export(void* hv, float* keys, float* values, uint8_t* text_code,
                         float* queries, float* centers, uint32_t* token_blob) {
    auto* h = static_cast<WorkloadH*>(hv);
    const auto& st = h->w.tokens;
    if (keys) std::memcpy(keys, st.keys_flat().data(), st.keys_flat().size_bytes());
    if (values) std::memcpy(values, st.values_flat().data(), st.values_flat().size_bytes());
    if (text_code)
        for (size_t i = 0; i < st.size(); ++i)
            text_code[i] = st.text(i).empty() ? 0 : (st.text(i) == "\n" ? 1 : 2);
    if (queries) std::memcpy(queries, h->w.queries.data(), h->w.queries.size() * 4);
    if (centers) std::memcpy(centers, h->w.blob_centers.data(), h->w.blob_centers.size() * 4);
    if (token_blob) std::memcpy(token_blob, h->w.token_blob.data(), h->w.token_blob.size() * 4);
}

// gen_local_queries (workload.cpp:171-190)
int tkr_local_queries(uint64_t n_tokens, uint64_t d, uint64_t n_blobs, double conc,
                      uint64_t seed, uint64_t blob, uint64_t count, uint64_t qseed,
                      float* out) {
    return guard([&] {
        WorkloadSpec s;
        s.n_tokens = n_tokens;
        s.d = d;
        s.n_blobs = n_blobs;
        s.blob_concentration = conc;
        s.seed = seed;
        auto q = gen_local_queries(s, blob, count, qseed);
        std::memcpy(out, q.data(), q.size() * 4);
    });
}

// splitmix64 + Box-Muller (workload.cpp:21-50); used to pin generator restatements
void tkr_rng_draws(uint64_t seed, uint64_t n_u64, uint64_t* u64_out, uint64_t n_gauss,
                   double* gauss_out) {
    Rng r(seed);
    for (uint64_t i = 0; i < n_u64; ++i) u64_out[i] = r.next_u64();
    Rng g(seed);
    for (uint64_t i = 0; i < n_gauss; ++i) gauss_out[i] = g.next_gaussian();
}

// ---- chunker (chunker.cpp:103-149) ---------------------------------------
// text codes as above; returns number of spans written (start,end,kind,level)
int tkr_segment(const uint8_t* text_code, uint64_t n, uint32_t* spans4, uint64_t cap,
                uint64_t* n_spans) {
    return guard([&] {
        std::vector<std::string> texts(n);
        for (uint64_t i = 0; i < n; ++i)
            texts[i] = text_code[i] == 1 ? "\n" : text_code[i] == 2 ? "}" : "";
        auto spans = segment(texts, ChunkPolicy::defaults());
        *n_spans = spans.size();
        for (size_t i = 0; i < spans.size() && i < cap; ++i) {
            spans4[4 * i + 0] = spans[i].start;
            spans4[4 * i + 1] = spans[i].end;
            spans4[4 * i + 2] = static_cast<uint32_t>(spans[i].kind);
            spans4[4 * i + 3] = static_cast<uint32_t>(spans[i].level);
        }
    });
}

// ---- engine = StreamState(store, build_index(store, spans, cfg)) ---------
// spans4 may be NULL: then the texts are segmented with ChunkPolicy::defaults()
int tkr_engine_new(const float* keys, const float* values, const uint8_t* text_code,
                   uint64_t n, uint64_t d, const uint32_t* spans4, uint64_t n_spans,
                   double avg_chunks, uint32_t max_units, uint32_t iters, uint32_t pooling,
                   uint64_t seed, uint32_t structure_aware, uint32_t graft_full,
                   void** out) {
    return guard([&] {
        TokenStore store = make_store(keys, values, text_code, n, d);
        std::vector<ChunkSpan> spans;
        if (spans4) {
            for (uint64_t i = 0; i < n_spans; ++i)
                spans.push_back({spans4[4 * i], spans4[4 * i + 1],
                                 static_cast<BoundaryKind>(spans4[4 * i + 2]),
                                 static_cast<int>(spans4[4 * i + 3])});
        } else {
            spans = segment(store.texts(), ChunkPolicy::defaults());
        }
        IndexConfig cfg;
        cfg.avg_chunks_per_cluster = avg_chunks;
        cfg.max_coarse_units = max_units;
        cfg.kmeans_iters = iters;
        cfg.pooling = pooling ? Pooling::max : Pooling::mean;
        cfg.seed = seed;
        HierarchicalIndex index = build_index(store, spans, cfg);
        StreamerConfig scfg;
        scfg.structure_aware = structure_aware != 0;
        scfg.graft_search = graft_full ? GraftSearch::full : GraftSearch::scoped;
        auto h = std::make_unique<EngineH>();
        h->state = std::make_unique<StreamState>(std::move(store), std::move(index), scfg);
        *out = h.release();
    });
}

void tkr_engine_free(void* h) { delete static_cast<EngineH*>(h); }

// dims[0..6] = dim, n_chunks, n_clusters, n_units, n_tokens, total fine members,
//              total coarse members ; dims[7] = buffer_size
void tkr_engine_dims(void* hv, uint64_t* dims) {
    const auto& st = *static_cast<EngineH*>(hv)->state;
    const auto& ix = st.index();
    dims[0] = ix.dim;
    dims[1] = ix.chunks.size();
    dims[2] = ix.fine.size();
    dims[3] = ix.coarse.size();
    dims[4] = st.store().size();
    size_t fm = 0, cm = 0;
    for (const auto& f : ix.fine) fm += f.members.size();
    for (const auto& c : ix.coarse) cm += c.members.size();
    dims[5] = fm;
    dims[6] = cm;
    dims[7] = st.buffer_size();
}

// Full export of the HierarchicalIndex (index.hpp:25-73) in its own numbering.
void tkr_engine_export(void* hv, uint32_t* chunk_span4, float* chunk_rep,
                       float* fine_centroid, double* fine_radius, uint64_t* fine_token_count,
                       uint32_t* fine_parent, uint32_t* fine_member_off, uint32_t* fine_members,
                       float* coarse_centroid, double* coarse_radius,
                       uint32_t* coarse_member_off, uint32_t* coarse_members,
                       uint32_t* cluster_of_chunk) {
    const auto& ix = static_cast<EngineH*>(hv)->state->index();
    const size_t d = ix.dim;
    for (size_t j = 0; j < ix.chunks.size(); ++j) {
        const auto& c = ix.chunks[j];
        if (chunk_span4) {
            chunk_span4[4 * j] = c.span.start;
            chunk_span4[4 * j + 1] = c.span.end;
            chunk_span4[4 * j + 2] = static_cast<uint32_t>(c.span.kind);
            chunk_span4[4 * j + 3] = static_cast<uint32_t>(c.span.level);
        }
        if (chunk_rep) std::memcpy(chunk_rep + j * d, c.rep_key.data(), d * 4);
    }
    uint32_t off = 0;
    for (size_t c = 0; c < ix.fine.size(); ++c) {
        const auto& f = ix.fine[c];
        if (fine_centroid) std::memcpy(fine_centroid + c * d, f.centroid.data(), d * 4);
        if (fine_radius) fine_radius[c] = f.radius;
        if (fine_token_count) fine_token_count[c] = f.token_count;
        if (fine_parent) fine_parent[c] = f.parent_unit;
        if (fine_member_off) fine_member_off[c] = off;
        if (fine_members) std::memcpy(fine_members + off, f.members.data(), f.members.size() * 4);
        off += static_cast<uint32_t>(f.members.size());
    }
    if (fine_member_off) fine_member_off[ix.fine.size()] = off;
    off = 0;
    for (size_t u = 0; u < ix.coarse.size(); ++u) {
        const auto& cu = ix.coarse[u];
        if (coarse_centroid) std::memcpy(coarse_centroid + u * d, cu.centroid.data(), d * 4);
        if (coarse_radius) coarse_radius[u] = cu.radius;
        if (coarse_member_off) coarse_member_off[u] = off;
        if (coarse_members)
            std::memcpy(coarse_members + off, cu.members.data(), cu.members.size() * 4);
        off += static_cast<uint32_t>(cu.members.size());
    }
    if (coarse_member_off) coarse_member_off[ix.coarse.size()] = off;
    if (cluster_of_chunk)
        std::memcpy(cluster_of_chunk, ix.cluster_of_chunk.data(), ix.cluster_of_chunk.size() * 4);
}

// index_to_bytes (serialize.cpp:88-125); returns the size, copies up to cap
uint64_t tkr_engine_index_bytes(void* hv, uint8_t* buf, uint64_t cap) {
    auto bytes = index_to_bytes(static_cast<EngineH*>(hv)->state->index());
    if (buf) std::memcpy(buf, bytes.data(), std::min<uint64_t>(cap, bytes.size()));
    return bytes.size();
}

// save_index (serialize.cpp:127-148) of the engine's index + store
int tkr_save_index(void* hv, const char* path) {
    return guard([&] { save_index(path, static_cast<EngineH*>(hv)->state->index()); });
}

// StreamState over load_index (serialize.cpp:150-220): a TKIX file written by
// either side becomes a reference engine
int tkr_engine_load(const char* path, uint32_t structure_aware, uint32_t graft_full, void** out) {
    return guard([&] {
        IndexFile f = load_index(path);
        StreamerConfig scfg;
        scfg.structure_aware = structure_aware != 0;
        scfg.graft_search = graft_full ? GraftSearch::full : GraftSearch::scoped;
        auto h = std::make_unique<EngineH>();
        h->state = std::make_unique<StreamState>(std::move(f.store), std::move(f.index), scfg);
        *out = h.release();
    });
}

// eval::oracle_topk_tokens (evaluator.cpp:43-64)
int tkr_oracle_topk(void* hv, const float* q, uint64_t d, uint64_t budget, uint32_t* out, uint64_t cap,
                    uint64_t* n) {
    return guard([&] {
        auto ids = eval::oracle_topk_tokens(std::span<const float>(q, d), static_cast<EngineH*>(hv)->state->store(),
                                            budget);
        copy_ids(ids, out, cap);
        *n = ids.size();
    });
}

void tkr_engine_store_export(void* hv, float* keys, float* values) {
    const auto& st = static_cast<EngineH*>(hv)->state->store();
    if (keys) std::memcpy(keys, st.keys_flat().data(), st.keys_flat().size_bytes());
    if (values) std::memcpy(values, st.values_flat().data(), st.values_flat().size_bytes());
}

// ---- retrieve / retrieve_ids (retriever.cpp:78-167) -----------------------
// counts[5] = n_units, n_clusters, n_active, scanned, degenerate
int tkr_retrieve(void* hv, const float* q, uint64_t d, uint32_t unit_topk, uint32_t mode,
                 uint32_t cluster_topk, uint64_t token_budget, uint32_t sink,
                 const uint32_t* buffer, uint64_t n_buffer, int with_output, uint32_t* units,
                 uint64_t units_cap, uint32_t* clusters, uint64_t clusters_cap,
                 uint32_t* active, uint64_t active_cap, float* output, uint64_t* counts) {
    return guard([&] {
        const auto& ix = static_cast<EngineH*>(hv)->state->index();
        Budgets b = make_budgets(unit_topk, mode, cluster_topk, token_budget, sink);
        std::span<const float> qs(q, d);
        std::span<const uint32_t> buf(buffer, n_buffer);
        RetrievalResult r = with_output ? retrieve(ix, qs, b, buf) : retrieve_ids(ix, qs, b, buf);
        write_result(r, units, units_cap, clusters, clusters_cap, active, active_cap, output,
                     counts);
    });
}

// sparse_attention (retriever.cpp:41-50) over an explicit id list
int tkr_sparse_attention(void* hv, const float* q, uint64_t d, const uint32_t* ids,
                         uint64_t n_ids, float* out) {
    return guard([&] {
        const auto& st = static_cast<EngineH*>(hv)->state->store();
        auto o = sparse_attention(std::span<const float>(q, d), st,
                                  std::span<const uint32_t>(ids, n_ids));
        std::memcpy(out, o.data(), o.size() * 4);
    });
}

// eval::full_attention (evaluator.cpp:11-41) over the engine's store
int tkr_full_attention(void* hv, const float* q, uint64_t d, float* out) {
    return guard([&] {
        const auto& st = static_cast<EngineH*>(hv)->state->store();
        auto o = eval::full_attention(std::span<const float>(q, d), st);
        std::memcpy(out, o.data(), o.size() * 4);
    });
}

// ---- streaming (streamer.cpp:145-165) -------------------------------------
// graft_out[8]: flag, chunk_id, cluster_id, unit_id, distance_comps (as double)
//               then centroid_delta, fine_radius, coarse_radius in graft_f64[3]
int tkr_decode_step(void* hv, const float* q, const float* key, const float* value,
                    uint8_t text_code, uint32_t unit_topk, uint32_t mode,
                    uint32_t cluster_topk, uint64_t token_budget, uint32_t sink,
                    uint32_t* units, uint64_t units_cap, uint32_t* clusters,
                    uint64_t clusters_cap, uint32_t* active, uint64_t active_cap,
                    float* output, uint64_t* counts, double* stab, uint64_t* graft_u,
                    double* graft_f64) {
    return guard([&] {
        auto& st = *static_cast<EngineH*>(hv)->state;
        const size_t d = st.store().dim();
        TokenRecord t;
        t.id = static_cast<uint32_t>(st.store().size());
        t.text = text_code == 1 ? "\n" : text_code == 2 ? "}" : "";
        t.key.assign(key, key + d);
        t.value.assign(value, value + d);
        Budgets b = make_budgets(unit_topk, mode, cluster_topk, token_budget, sink);
        DecodeOutcome o = st.decode_step(std::span<const float>(q, d), t, b);
        write_result(o.retrieval, units, units_cap, clusters, clusters_cap, active, active_cap,
                     output, counts);
        if (stab) {
            stab[0] = o.jaccard;
            stab[1] = o.window_hit;
        }
        if (graft_u) {
            graft_u[0] = o.graft ? 1 : 0;
            if (o.graft) {
                graft_u[1] = o.graft->chunk_id;
                graft_u[2] = o.graft->cluster_id;
                graft_u[3] = o.graft->unit_id;
                graft_u[4] = o.graft->distance_comps;
                const auto& c = st.index().chunks.back();
                graft_u[5] = c.span.start;
                graft_u[6] = c.span.end;
            }
        }
        if (graft_f64 && o.graft) {
            graft_f64[0] = o.graft->centroid_delta;
            graft_f64[1] = o.graft->fine_radius;
            graft_f64[2] = o.graft->coarse_radius;
        }
    });
}

// push_token + graft_chunk as two separate reference calls (streamer.cpp:56-143)
int tkr_push_and_graft(void* hv, const float* key, const float* value, uint8_t text_code,
                       uint64_t* graft_u, double* graft_f64) {
    return guard([&] {
        auto& st = *static_cast<EngineH*>(hv)->state;
        const size_t d = st.store().dim();
        TokenRecord t;
        t.id = static_cast<uint32_t>(st.store().size());
        t.text = text_code == 1 ? "\n" : text_code == 2 ? "}" : "";
        t.key.assign(key, key + d);
        t.value.assign(value, value + d);
        auto chunk = st.push_token(t);
        graft_u[0] = chunk ? 1 : 0;
        if (chunk) {
            auto r = st.graft_chunk(std::move(*chunk));
            graft_u[1] = r.chunk_id;
            graft_u[2] = r.cluster_id;
            graft_u[3] = r.unit_id;
            graft_u[4] = r.distance_comps;
            graft_f64[0] = r.centroid_delta;
            graft_f64[1] = r.fine_radius;
            graft_f64[2] = r.coarse_radius;
        }
    });
}

// chunk_representative (index.cpp:20-41)
int tkr_chunk_representative(const float* keys, uint64_t rows, uint64_t d, uint32_t pooling,
                             float* out) {
    return guard([&] {
        auto r = chunk_representative(std::span<const float>(keys, rows * d), d,
                                      pooling ? Pooling::max : Pooling::mean);
        std::memcpy(out, r.data(), d * 4);
    });
}

// audit_ub_soundness (evaluator.cpp:107-140)
uint64_t tkr_audit(void* hv, const float* queries, uint64_t nq, double tol) {
    const auto& ix = static_cast<EngineH*>(hv)->state->index();
    return eval::audit_ub_soundness(ix, std::span<const float>(queries, nq * ix.dim), nq, tol);
}

// ---- CPU timing of the reference hot path ---------------------------------
// Runs retrieve() (ids + sparse attention, the reference's own stock path)
// for every (engine e, query i) with q = queries[(e*nq_per + i)*d], `reps`
// times, and returns the wall seconds of the whole loop.  mode 0 = the
// reference API as-is (serial over calls, OpenMP inside the kernels);
// mode 1 = OpenMP over calls with single-threaded kernels (nested disabled).
double tkr_time_retrieve(void** engines, uint64_t n_eng, const float* queries, uint64_t nq_per,
                         uint64_t d, uint32_t unit_topk, uint64_t token_budget, uint32_t sink,
                         uint32_t reps, int mode, int threads, uint64_t* checksum_active) {
    Budgets b = make_budgets(unit_topk, 1, 8, token_budget, sink);
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    const uint64_t total = n_eng * nq_per;
    uint64_t acc = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (uint32_t r = 0; r < reps; ++r) {
        if (mode == 0) {
            for (uint64_t c = 0; c < total; ++c) {
                const auto& ix = static_cast<EngineH*>(engines[c / nq_per])->state->index();
                auto res = retrieve(ix, std::span<const float>(queries + c * d, d), b);
                acc += res.active_token_ids.size();
            }
        } else {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : acc)
#endif
            for (uint64_t c = 0; c < total; ++c) {
                const auto& ix = static_cast<EngineH*>(engines[c / nq_per])->state->index();
                auto res = retrieve(ix, std::span<const float>(queries + c * d, d), b);
                acc += res.active_token_ids.size();
            }
        }
    }
    auto t1 = std::chrono::steady_clock::now();
    if (checksum_active) *checksum_active = acc;
    return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
