// Per-call latency of the reference's own C++ API on its hot path --
// tierkv::retrieve() (retriever.cpp:161-167) and StreamState::decode_step()
// (streamer.cpp:145-165) -- for one (layer, KV head) slot, built from the
// reference's gen_clustered_workload + build_index.  The same source links
// twice (oracle/Makefile): against the reference library (CPU, its OpenMP
// kernels on every host thread) and against the B200 drop-in
// (paper_2603_08453_b200/cpp/tierkv_dropin.cpp over the C ABI), so the two
// binaries time the same calls a reference user makes.
//
//   dropin_bench <n_tokens> <queries> <decode_steps>   -> one JSON line
#include "tierkv/index.hpp"
#include "tierkv/retriever.hpp"
#include "tierkv/streamer.hpp"
#include "tierkv/chunker.hpp"
#include "tierkv/workload.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace tierkv;
using clk = std::chrono::steady_clock;

static double pct(std::vector<double> v, double p) {
    std::sort(v.begin(), v.end());
    return v[std::min(v.size() - 1, (size_t)(p * (v.size() - 1) + 0.5))];
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 32768;
    const size_t nq = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 64;
    const size_t steps = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 256;
    WorkloadSpec spec;
    spec.n_tokens = n;
    spec.d = 128;
    spec.query_count = nq;
    spec.seed = 1000;
    auto t0 = clk::now();
    Workload w = gen_clustered_workload(spec);
    auto spans = segment(w.tokens.texts(), ChunkPolicy::defaults());
    IndexConfig icfg;
    icfg.seed = spec.seed;
    HierarchicalIndex index = build_index(w.tokens, spans, icfg);
    const double build_s = std::chrono::duration<double>(clk::now() - t0).count();
    Budgets b;
    b.token_budget = 2048;
    const size_t d = spec.d;

    // retrieve(): first call (device engine creation + upload on the drop-in)
    // then nq timed calls with distinct queries against the same index
    auto tf = clk::now();
    auto r0 = retrieve(index, std::span<const float>(w.queries.data(), d), b);
    const double first_ms = std::chrono::duration<double, std::milli>(clk::now() - tf).count();
    std::vector<double> lat;
    size_t acc = r0.active_token_ids.size();
    for (size_t i = 0; i < nq; ++i) {
        auto a = clk::now();
        auto r = retrieve(index, std::span<const float>(w.queries.data() + (i % nq) * d, d), b);
        lat.push_back(std::chrono::duration<double, std::micro>(clk::now() - a).count());
        acc += r.active_token_ids.size();
    }

    // decode_step(): run_stream-style stationary decode (bench.cpp:240-272)
    StreamerConfig scfg;
    StreamState state(std::move(w.tokens), std::move(index), scfg);
    Rng rng(7);
    const float* center = w.blob_centers.data();
    std::vector<double> dlat;
    size_t grafts = 0;
    for (size_t s = 0; s < steps; ++s) {
        std::vector<float> q(d);
        double n2 = 0;
        for (size_t j = 0; j < d; ++j) {
            q[j] = static_cast<float>(center[j] + 0.33 / std::sqrt((double)d) * rng.next_gaussian());
            n2 += (double)q[j] * q[j];
        }
        for (auto& x : q) x = static_cast<float>(x * std::sqrt((double)d / n2));
        TokenRecord tok;
        tok.id = static_cast<uint32_t>(state.store().size());
        if ((s + 1) % 12 == 0) tok.text = "\n";
        tok.key.resize(d);
        double k2 = 0;
        for (size_t j = 0; j < d; ++j) {
            tok.key[j] = static_cast<float>(center[j] + 0.33 / std::sqrt((double)d) * rng.next_gaussian());
            k2 += (double)tok.key[j] * tok.key[j];
        }
        for (auto& x : tok.key) x = static_cast<float>(x / std::sqrt(k2));
        tok.value.resize(d);
        for (auto& x : tok.value) x = static_cast<float>(rng.next_gaussian());
        auto a = clk::now();
        auto out = state.decode_step(q, tok, b);
        dlat.push_back(std::chrono::duration<double, std::micro>(clk::now() - a).count());
        grafts += out.graft.has_value();
    }
    double rmean = 0, dmean = 0;
    for (double x : lat) rmean += x;
    for (double x : dlat) dmean += x;
    rmean /= std::max<size_t>(1, lat.size());
    dmean /= std::max<size_t>(1, dlat.size());
    std::printf(
        "{\"n_tokens\": %zu, \"build_s\": %.2f, \"retrieve_first_ms\": %.3f, \"retrieve_us\": {\"mean\": %.1f, "
        "\"p50\": %.1f, \"p90\": %.1f, \"calls\": %zu}, \"decode_step_us\": {\"mean\": %.1f, \"p50\": %.1f, "
        "\"p90\": %.1f, \"steps\": %zu, \"grafts\": %zu}, \"checksum_active\": %zu}\n",
        n, build_s, first_ms, rmean, pct(lat, 0.5), pct(lat, 0.9), lat.size(), dmean, pct(dlat, 0.5),
        pct(dlat, 0.9), dlat.size(), grafts, acc);
    return 0;
}
