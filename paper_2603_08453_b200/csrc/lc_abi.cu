// Host side of the C ABI (include/lychee_b200.h): the engine arena, slot
// upload/download in the reference's numbering, and the stream-ordered
// launch sequence of every decode-step operation.  No exception crosses the
// ABI; every entry point returns an LC_* status and records lc_last_error().
#include "../../include/lychee_b200.h"
#include "lc_common.cuh"


#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lc_engine.hpp"

static uint32_t needed_candidates(lc_index_s* h, uint32_t unit_topk) {
    auto it = h->cand_cache.find(unit_topk);
    if (it != h->cand_cache.end()) return it->second;
    uint32_t best = 1;
    for (const auto& s : h->hs) {
        if (!s.loaded) continue;
        std::vector<uint32_t> f = s.fanout;
        std::sort(f.begin(), f.end(), std::greater<uint32_t>());
        uint64_t sum = 0;
        for (size_t i = 0; i < f.size() && i < unit_topk; ++i) sum += f[i];
        best = std::max<uint32_t>(best, (uint32_t)std::min<uint64_t>(sum, 0xffffffffu));
    }
    h->cand_cache[unit_topk] = best;
    return best;
}

// lc_decode_step_async leaves the host's per-slot cursors behind the device:
// re-read them (and the grafted chunks' kind / level) before a host-side call
void sync_host(lc_index_t h) {
    if (!h || !h->dev_ahead) return;
    h->set_device();
    ck(cudaDeviceSynchronize(), "sync");
    const Arena& a = h->a;
    std::vector<SlotState> st(a.n_slots);
    ck(cudaMemcpy(st.data(), a.state, st.size() * sizeof(SlotState), cudaMemcpyDeviceToHost), "state");
    std::vector<uint32_t> kl;
    for (uint32_t s = 0; s < a.n_slots; ++s) {
        HostSlot& hs = h->hs[s];
        if (!hs.loaded) continue;
        if (st[s].n_chunks > hs.n_chunks) {
            kl.resize(st[s].n_chunks - hs.n_chunks);
            ck(cudaMemcpy(kl.data(), a.chunk_kl + (size_t)s * a.cap_chunks + hs.n_chunks, kl.size() * 4,
                          cudaMemcpyDeviceToHost), "chunk kinds");
            for (uint32_t v : kl) {
                hs.kind.push_back(v & 0xffu);
                hs.level.push_back(v >> 8);
            }
            if (!hs.rep.empty()) hs.rep.clear();  // prefill reps no longer complete
        }
        hs.n_tokens = st[s].n_tokens;
        hs.chunked_end = st[s].chunked_end;
        hs.n_chunks = st[s].n_chunks;
    }
    h->dev_ahead = false;
}

extern "C" {

const char* lc_last_error(void) { return g_err.c_str(); }

int lc_index_create(const lc_index_desc* desc, lc_index_t* out) {
    return guard([&] {
        if (!desc || !out) fail(LC_EINVAL, "lc_index_create: null argument");
        const lc_index_desc& d = *desc;
        if (d.n_slots == 0 || d.dim == 0 || d.group == 0 || d.group > (uint32_t)kMaxGroup)
            fail(LC_EINVAL, "lc_index_create: need n_slots >= 1, dim >= 1, 1 <= group <= 8");
        if (d.kv_f32 > 1) fail(LC_EINVAL, "lc_index_create: kv_f32 must be 0 or 1");
        // head dims with compiled kernels: 64/128 for every group size; the
        // reference-exact fp32 mode adds 8/16/32 for single-head and GQA-4 slots
        const bool big = d.dim == 64 || d.dim == 128;
        const bool small = (d.dim == 8 || d.dim == 16 || d.dim == 32) && d.kv_f32 && (d.group == 1 || d.group == 4);
        if (!big && !small)
            fail(LC_EINVAL, "lc_index_create: dim must be 64 or 128 (or 8/16/32 with kv_f32 and group 1 or 4)");
        if (d.cap_units == 0 || d.cap_units > 1024) fail(LC_EINVAL, "lc_index_create: 1 <= cap_units <= 1024");
        if (d.cap_tokens == 0 || d.cap_chunks == 0 || d.cap_clusters == 0)
            fail(LC_EINVAL, "lc_index_create: zero capacity");
        if (d.cap_tokens >= (1u << 24)) fail(LC_EINVAL, "lc_index_create: cap_tokens must be < 2^24");
        if (d.group != 1 && d.group != 2 && d.group != 4 && d.group != 8)
            fail(LC_EINVAL, "lc_index_create: group must be 1, 2, 4 or 8");
        // k_coarse stages the coarse tier [d][P] and G x P keys in shared memory
        const uint32_t cu4 = (d.cap_units + 3) & ~3u;
        if ((size_t)d.dim * cu4 * 4 > 96 * 1024 || (size_t)d.group * cu4 > 1024)
            fail(LC_EINVAL, "lc_index_create: cap_units too large for the coarse-tier kernel "
                            "(need dim*cap_units*4 <= 96 KiB and group*cap_units <= 1024)");
        auto h = std::make_unique<lc_index_s>();
        h->desc = d;
        h->kv_elem = d.kv_f32 ? 4u : 2u;
        h->set_device();
        Arena& a = h->a;
        a.n_slots = d.n_slots;
        a.d = d.dim;
        a.G = d.group;
        a.cap_tokens = d.cap_tokens;
        a.cap_chunks = d.cap_chunks;
        a.cap_clusters = d.cap_clusters;
        a.cap_units = (d.cap_units + 3) & ~3u;  // float4 rows of the coarse tier
        a.max_cand = 1;
        a.graft_full = d.graft_full;
        a.keep_reps = d.keep_reps;
        a.kv_f32 = d.kv_f32;
        a.cap_spans = d.cap_chunks + 2 + 1024;
        const size_t S = d.n_slots, D = d.dim, G = d.group;
        auto& o = h->owned;
        if (d.kv_f32) {
            a.Kf = dalloc<float>(S * d.cap_tokens * D, o);
            a.Vf = dalloc<float>(S * d.cap_tokens * D, o);
        } else {
            a.K = dalloc<__nv_bfloat16>(S * d.cap_tokens * D, o);
            a.V = dalloc<__nv_bfloat16>(S * d.cap_tokens * D, o);
        }
        a.chunk_start = dalloc<uint32_t>(S * (d.cap_chunks + 1), o);
        a.chunk_clu = dalloc<uint32_t>(S * d.cap_chunks, o);
        a.chunk_rep = d.keep_reps ? dalloc<float>(S * d.cap_chunks * D, o) : nullptr;
        a.ucent = dalloc<float>(S * a.cap_units * D, o);
        a.urad = dalloc<double>(S * a.cap_units, o);
        a.unit_off = dalloc<uint32_t>(S * (a.cap_units + 1), o);
        a.fcent = dalloc<float>(S * d.cap_clusters * D, o);
        a.frow16 = dalloc<__half>(S * d.cap_clusters * D, o);
        a.fmeta = dalloc<uint4>(S * d.cap_clusters, o);
        a.frad = dalloc<double>(S * d.cap_clusters, o);
        a.ftok = dalloc<uint32_t>(S * d.cap_clusters, o);
        a.forig = dalloc<uint32_t>(S * d.cap_clusters, o);
        a.fnmem = dalloc<uint32_t>(S * d.cap_clusters, o);
        a.funit = dalloc<uint32_t>(S * d.cap_clusters, o);
        a.fmem_off = dalloc<uint32_t>(S * (d.cap_clusters + 1), o);
        a.fmem = dalloc<uint32_t>(S * d.cap_chunks, o);
        a.chunk_kl = dalloc<uint32_t>(S * d.cap_chunks, o);
        a.plan_bytes = plan_layout(a.cap_units, d.group, d.dim, d.cap_clusters, nullptr, nullptr, nullptr);
        a.plan = dalloc<unsigned char>(S * a.plan_bytes, o);
        a.chunk_bits = dalloc<uint32_t>(S * G * bit_words(d.cap_chunks), o);
        a.state = dalloc<SlotState>(S, o);
        a.qinfo = dalloc<QInfo>(S * G, o);
        a.sel_units = dalloc<uint32_t>(S * G * a.cap_units, o);
        a.sel_clusters = dalloc<uint32_t>(S * G * d.cap_clusters, o);
        a.sel_bits = dalloc<uint32_t>(S * G * bit_words(d.cap_clusters), o);
        a.spans = dalloc<Span>(S * a.cap_spans, o);
        a.span_off = dalloc<uint32_t>(S * (a.cap_spans + 1), o);
        a.n_spans = dalloc<uint32_t>(S, o);
        a.rows = dalloc<uint32_t>(S * d.cap_tokens, o);
        a.slot_tok = dalloc<uint32_t>(S, o);
        a.step_bytes = dalloc<unsigned long long>(S * 4, o);
        // attention partials + the persistent kernel's pool / barrier counters (zeroed)
        const size_t part_floats = attend_partials_floats(a.d, a.G, a.n_slots);
        h->att_part = dalloc<float>(part_floats, o);
        ck(cudaMemset(h->att_part, 0, part_floats * 4), "memset attention partials");
        const size_t groups = std::max<uint32_t>(1, std::min(d.slot_groups, d.n_slots));
        h->fine_ctr = dalloc<uint32_t>(32 * groups, o);
        ck(cudaMemset(h->fine_ctr, 0, 32 * groups * 4), "memset k_fine / k_pickq counters");
        h->pick_ord = dalloc<uint32_t>((size_t)16 * S * G, o);
        a.err = dalloc<uint32_t>(1, o);
        h->q_stage = dalloc<float>(S * G * D, o);
        h->out_stage = dalloc<float>(S * G * D, o);
        h->take_dev = dalloc<uint32_t>(S, o);
        h->rep_scratch = dalloc<lc_graft_report>(S, o);
        h->reps_dev = dalloc<float>(S * D, o);
        ck(cudaMemset(a.state, 0, S * sizeof(SlotState)), "memset state");
        ck(cudaMemset(a.err, 0, 4), "memset err");
        ck(cudaMemset(a.n_spans, 0, S * 4), "memset n_spans");
        ck(cudaMemset(a.slot_tok, 0, S * 4), "memset slot_tok");
        ck(cudaMemset(a.span_off, 0, S * (a.cap_spans + 1) * 4), "memset span_off");
        ck(cudaMemset(a.qinfo, 0, S * G * sizeof(QInfo)), "memset qinfo");
        h->hs.resize(S);
        *out = h.release();
    });
}

void lc_index_destroy(lc_index_t h) {
    if (!h) return;
    cudaSetDevice(h->desc.device);
    cudaDeviceSynchronize();
    delete h;
}

int lc_index_get_desc(lc_index_t h, lc_index_desc* out) {
    return guard([&] {
        if (!h || !out) fail(LC_EINVAL, "null argument");
        *out = h->desc;
    });
}

int lc_index_upload_slot(lc_index_t h, uint32_t slot, const lc_host_index* ix,
                         const void* keys, const void* values, uint32_t n_tokens) {
    return guard([&] {
        if (!h || !ix) fail(LC_EINVAL, "lc_index_upload_slot: null argument");
        sync_host(h);
        h->set_device();
        const Arena& a = h->a;
        if (slot >= a.n_slots) fail(LC_EINVAL, "slot out of range");
        const uint32_t D = a.d, M = ix->n_chunks, L = ix->n_clusters, P = ix->n_units;
        if (ix->dim != D) fail(LC_EINVAL, "index dimension mismatch");
        if (L == 0) fail(LC_EINVAL, "stream state: empty index");  // streamer.cpp:16
        if (n_tokens > a.cap_tokens || M > a.cap_chunks || L > a.cap_clusters || P > a.cap_units || P == 0)
            fail(LC_EINVAL, "slot exceeds engine capacity");
        // chunks must tile [0, chunked_end) (build_index, index.cpp:160-167)
        uint32_t expect = 0;
        for (uint32_t j = 0; j < M; ++j) {
            const uint32_t s = ix->chunk_span[4 * j], e = ix->chunk_span[4 * j + 1];
            if (s != expect || e <= s) fail(LC_EINVAL, "chunks do not tile the stream");
            expect = e;
        }
        const uint32_t chunked_end = expect;
        if (chunked_end > n_tokens) fail(LC_EINVAL, "stream state: chunks exceed store");
        // internal renumbering: coarse members concatenated in unit order
        std::vector<uint32_t> int_of(L, 0xffffffffu), orig(L), unit_off(P + 1);
        uint32_t pos = 0;
        for (uint32_t u = 0; u < P; ++u) {
            unit_off[u] = pos;
            for (uint32_t m = ix->coarse_member_off[u]; m < ix->coarse_member_off[u + 1]; ++m) {
                const uint32_t f = ix->coarse_members[m];
                if (f >= L || int_of[f] != 0xffffffffu) fail(LC_EINVAL, "coarse members are not a partition");
                if (ix->fine_parent[f] != u) fail(LC_EINVAL, "fine parent_unit disagrees with coarse members");
                int_of[f] = pos;
                orig[pos++] = f;
            }
        }
        unit_off[P] = pos;
        if (pos != L) fail(LC_EINVAL, "coarse members do not cover every fine cluster");
        // cluster_of_chunk must agree with the fine member lists
        std::vector<uint32_t> nmem(L, 0);
        for (uint32_t f = 0; f < L; ++f)
            for (uint32_t m = ix->fine_member_off[f]; m < ix->fine_member_off[f + 1]; ++m) {
                const uint32_t j = ix->fine_members[m];
                if (j >= M || ix->cluster_of_chunk[j] != f) fail(LC_EINVAL, "fine members disagree with cluster_of_chunk");
                ++nmem[f];
            }
        std::vector<float> fcent((size_t)L * D), ucent((size_t)a.cap_units * D, 0.f);
        std::vector<__half> f16((size_t)L * D);  // the filters' copy; their error bound needs |c| <= 6e4
        std::vector<double> cn2(L, 0.0);
        std::vector<double> frad(L), urad(P);
        std::vector<uint32_t> ftok(L), fn(L), fu(L);
        for (uint32_t u = 0; u < P; ++u) {
            const uint32_t base = unit_off[u], nu = unit_off[u + 1] - base;
            for (uint32_t i = 0; i < nu; ++i) {
                const uint32_t f = orig[base + i];
                for (uint32_t j = 0; j < D; ++j) {
                    const float c = ix->fine_centroid[(size_t)f * D + j];
                    if (!(std::fabs(c) <= 60000.f)) fail(LC_EINVAL, "fine centroids must be finite and |c| <= 6e4");
                    fcent[fine_at(base, nu, i, j, D)] = c;
                    f16[frow_at(base, i, j, D)] = __float2half_rn(c);
                    cn2[base + i] += (double)c * (double)c;
                }
            }
            for (uint32_t j = 0; j < D; ++j) ucent[(size_t)j * a.cap_units + u] = ix->coarse_centroid[(size_t)u * D + j];
            urad[u] = ix->coarse_radius[u];
        }
        std::vector<uint4> meta(L);
        float rmax = 0.f, cmax = 0.f;
        for (uint32_t i = 0; i < L; ++i) {
            const uint32_t f = orig[i];
            frad[i] = ix->fine_radius[f];
            if (!(frad[i] >= 0.0 && frad[i] < 1e30)) fail(LC_EINVAL, "fine radii must be finite and >= 0");
            if (ix->fine_token_count[f] > 0xffffffffull) fail(LC_EINVAL, "token_count exceeds u32");
            ftok[i] = (uint32_t)ix->fine_token_count[f];
            fn[i] = nmem[f];
            fu[i] = ix->fine_parent[f];
            uint64_t rb;
            std::memcpy(&rb, &frad[i], 8);
            const float cb = norm_bound(cn2[i]);
            uint32_t cbits;
            std::memcpy(&cbits, &cb, 4);
            meta[i] = make_uint4((uint32_t)rb, (uint32_t)(rb >> 32), cbits, ftok[i]);
            float rf = (float)frad[i];
            if ((double)rf < frad[i]) rf = nextafterf(rf, 3.0e38f);
            rmax = std::max(rmax, rf);
            cmax = std::max(cmax, cb);
        }
        std::vector<uint32_t> cs(M + 1), cc(M);
        for (uint32_t j = 0; j < M; ++j) {
            cs[j] = ix->chunk_span[4 * j];
            cc[j] = int_of[ix->cluster_of_chunk[j]];
        }
        cs[M] = chunked_end;
        // member CSR by internal cluster id, chunk ids ascending
        std::vector<uint32_t> moff(L + 1, 0), mem(M);
        for (uint32_t j = 0; j < M; ++j) ++moff[cc[j] + 1];
        for (uint32_t c = 0; c < L; ++c) moff[c + 1] += moff[c];
        {
            std::vector<uint32_t> cur(moff.begin(), moff.end() - 1);
            for (uint32_t j = 0; j < M; ++j) mem[cur[cc[j]]++] = j;
        }
        const size_t so = slot;
        auto up = [&](void* dst, const void* src, size_t bytes) {
            if (bytes) ck(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "upload");
        };
        if (keys) up(h->kv_ptr(0, slot), keys, (size_t)n_tokens * D * h->kv_elem);
        if (values) up(h->kv_ptr(1, slot), values, (size_t)n_tokens * D * h->kv_elem);
        up(a.chunk_start + so * (a.cap_chunks + 1), cs.data(), cs.size() * 4);
        up(a.chunk_clu + so * a.cap_chunks, cc.data(), cc.size() * 4);
        up(a.ucent + so * a.cap_units * D, ucent.data(), ucent.size() * 4);
        up(a.urad + so * a.cap_units, urad.data(), urad.size() * 8);
        up(a.unit_off + so * (a.cap_units + 1), unit_off.data(), unit_off.size() * 4);
        up(a.fcent + so * a.cap_clusters * D, fcent.data(), fcent.size() * 4);
        up(a.frow16 + so * a.cap_clusters * D, f16.data(), f16.size() * 2);
        up(a.fmeta + so * a.cap_clusters, meta.data(), meta.size() * 16);
        up(a.frad + so * a.cap_clusters, frad.data(), frad.size() * 8);
        up(a.ftok + so * a.cap_clusters, ftok.data(), ftok.size() * 4);
        up(a.forig + so * a.cap_clusters, orig.data(), orig.size() * 4);
        up(a.fnmem + so * a.cap_clusters, fn.data(), fn.size() * 4);
        up(a.funit + so * a.cap_clusters, fu.data(), fu.size() * 4);
        up(a.fmem_off + so * (a.cap_clusters + 1), moff.data(), moff.size() * 4);
        up(a.fmem + so * a.cap_chunks, mem.data(), mem.size() * 4);
        HostSlot& hs = h->hs[slot];
        hs = HostSlot{};
        hs.cfg.pooling = h->desc.pooling;
        hs.kind.resize(M);
        hs.level.resize(M);
        for (uint32_t j = 0; j < M; ++j) {
            hs.kind[j] = ix->chunk_span[4 * j + 2];
            hs.level[j] = ix->chunk_span[4 * j + 3];
        }
        if (ix->chunk_rep) {
            if (a.keep_reps) up(a.chunk_rep + so * a.cap_chunks * D, ix->chunk_rep, (size_t)M * D * 4);
            else hs.rep.assign(ix->chunk_rep, ix->chunk_rep + (size_t)M * D);
        }
        SlotState st{};
        st.n_tokens = n_tokens;
        st.chunked_end = chunked_end;
        st.n_chunks = M;
        st.m0 = M;
        st.L = L;
        st.P = P;
        st.rmax = rmax;
        st.cmax = cmax;
        up(a.state + slot, &st, sizeof st);
        hs.n_tokens = n_tokens;
        hs.chunked_end = chunked_end;
        hs.n_chunks = M;
        hs.L = L;
        hs.P = P;
        hs.loaded = true;
        hs.fanout.resize(P);
        for (uint32_t u = 0; u < P; ++u) hs.fanout[u] = unit_off[u + 1] - unit_off[u];
        h->cand_cache.clear();
        ++h->version;
    });
}

int lc_index_slot_dims(lc_index_t h, uint32_t slot, uint64_t* dims) {
    return guard([&] {
        if (!h || !dims || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_index_slot_dims: bad argument");
        sync_host(h);
        const HostSlot& s = h->hs[slot];
        dims[0] = h->a.d;
        dims[1] = s.n_chunks;
        dims[2] = s.L;
        dims[3] = s.P;
        dims[4] = s.n_tokens;
        dims[5] = s.n_chunks;  // every chunk belongs to exactly one cluster
        dims[6] = s.L;         // every cluster belongs to exactly one unit
        dims[7] = s.chunked_end;
    });
}

int lc_index_download_slot(lc_index_t h, uint32_t slot, lc_host_index* ix) {
    return guard([&] {
        if (!h || !ix || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_index_download_slot: bad argument");
        sync_host(h);
        h->set_device();
        ck(cudaDeviceSynchronize(), "sync");
        const Arena& a = h->a;
        const HostSlot& hs = h->hs[slot];
        const uint32_t D = a.d, M = hs.n_chunks, L = hs.L, P = hs.P;
        const size_t so = slot;
        auto down = [&](void* dst, const void* src, size_t bytes) {
            if (bytes) ck(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "download");
        };
        SlotState st;
        down(&st, a.state + slot, sizeof st);
        if (st.n_chunks != M || st.n_tokens != hs.n_tokens || st.chunked_end != hs.chunked_end)
            fail(LC_ERUNTIME, "device and host stream cursors diverged");
        std::vector<uint32_t> cs(M + 1), cc(M), unit_off(P + 1), orig(L), ftok(L), fu(L);
        std::vector<float> fcent((size_t)L * D), ucent((size_t)a.cap_units * D);
        std::vector<double> frad(L), urad(P);
        down(cs.data(), a.chunk_start + so * (a.cap_chunks + 1), cs.size() * 4);
        down(cc.data(), a.chunk_clu + so * a.cap_chunks, cc.size() * 4);
        down(unit_off.data(), a.unit_off + so * (a.cap_units + 1), unit_off.size() * 4);
        down(orig.data(), a.forig + so * a.cap_clusters, orig.size() * 4);
        down(ftok.data(), a.ftok + so * a.cap_clusters, ftok.size() * 4);
        down(fu.data(), a.funit + so * a.cap_clusters, fu.size() * 4);
        down(fcent.data(), a.fcent + so * a.cap_clusters * D, fcent.size() * 4);
        down(ucent.data(), a.ucent + so * a.cap_units * D, ucent.size() * 4);
        down(frad.data(), a.frad + so * a.cap_clusters, frad.size() * 8);
        down(urad.data(), a.urad + so * a.cap_units, urad.size() * 8);
        ix->dim = D;
        ix->n_chunks = M;
        ix->n_clusters = L;
        ix->n_units = P;
        for (uint32_t j = 0; j < M; ++j) {
            ix->chunk_span[4 * j] = cs[j];
            ix->chunk_span[4 * j + 1] = cs[j + 1];
            ix->chunk_span[4 * j + 2] = hs.kind[j];
            ix->chunk_span[4 * j + 3] = hs.level[j];
            ix->cluster_of_chunk[j] = orig[cc[j]];
        }
        if (ix->chunk_rep) {
            if (a.keep_reps) down(ix->chunk_rep, a.chunk_rep + so * a.cap_chunks * D, (size_t)M * D * 4);
            else if (hs.rep.size() == (size_t)M * D) std::memcpy(ix->chunk_rep, hs.rep.data(), hs.rep.size() * 4);
            else recompute_slot_reps(h, slot, cs.data(), M, ix->chunk_rep);
        }
        for (uint32_t u = 0; u < P; ++u) {
            const uint32_t base = unit_off[u], nu = unit_off[u + 1] - base;
            for (uint32_t i = 0; i < nu; ++i) {
                const uint32_t f = orig[base + i];
                for (uint32_t j = 0; j < D; ++j)
                    ix->fine_centroid[(size_t)f * D + j] = fcent[fine_at(base, nu, i, j, D)];
            }
            for (uint32_t j = 0; j < D; ++j) ix->coarse_centroid[(size_t)u * D + j] = ucent[(size_t)j * a.cap_units + u];
            ix->coarse_radius[u] = urad[u];
            ix->coarse_member_off[u] = base;
            for (uint32_t i = 0; i < nu; ++i) ix->coarse_members[base + i] = orig[base + i];
        }
        ix->coarse_member_off[P] = unit_off[P];
        for (uint32_t i = 0; i < L; ++i) {
            const uint32_t f = orig[i];
            ix->fine_radius[f] = frad[i];
            ix->fine_token_count[f] = ftok[i];
            ix->fine_parent[f] = fu[i];
        }
        // fine member lists: ascending chunk ids per cluster (build order, then grafts)
        std::vector<uint32_t> cnt(L + 1, 0);
        for (uint32_t j = 0; j < M; ++j) ++cnt[ix->cluster_of_chunk[j] + 1];
        for (uint32_t f = 0; f < L; ++f) cnt[f + 1] += cnt[f];
        for (uint32_t f = 0; f <= L; ++f) ix->fine_member_off[f] = cnt[f];
        for (uint32_t j = 0; j < M; ++j) ix->fine_members[cnt[ix->cluster_of_chunk[j]]++] = j;
    });
}

int lc_cluster_download(lc_index_t h, uint32_t slot, uint32_t cluster_id, float* centroid, double* radius,
                        uint64_t* token_count) {
    return guard([&] {
        if (!h || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_cluster_download: bad argument");
        sync_host(h);
        HostSlot& hs = h->hs[slot];
        if (!hs.loaded || cluster_id >= hs.L) fail(LC_EINVAL, "lc_cluster_download: no such cluster");
        h->set_device();
        const Arena& a = h->a;
        if (hs.internal_of.size() != hs.L) {  // the renumbering is fixed once a slot is uploaded / built
            std::vector<uint32_t> orig(hs.L);
            ck(cudaMemcpy(orig.data(), a.forig + (size_t)slot * a.cap_clusters, hs.L * 4, cudaMemcpyDeviceToHost),
               "forig");
            hs.internal_of.assign(hs.L, 0);
            for (uint32_t i = 0; i < hs.L; ++i) hs.internal_of[orig[i]] = i;
        }
        const size_t c = (size_t)slot * a.cap_clusters + hs.internal_of[cluster_id];
        ck(cudaDeviceSynchronize(), "sync");
        if (centroid) ck(cudaMemcpy(centroid, a.fcent + c * a.d, (size_t)a.d * 4, cudaMemcpyDeviceToHost), "centroid");
        if (radius) ck(cudaMemcpy(radius, a.frad + c, 8, cudaMemcpyDeviceToHost), "radius");
        if (token_count) {
            uint32_t t = 0;
            ck(cudaMemcpy(&t, a.ftok + c, 4, cudaMemcpyDeviceToHost), "token count");
            *token_count = t;
        }
    });
}

int lc_kv_upload_slot(lc_index_t h, uint32_t slot, const void* keys, const void* values,
                      uint32_t n_tokens) {
    return guard([&] {
        if (!h || !keys || !values || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_kv_upload_slot: bad argument");
        sync_host(h);
        if (n_tokens > h->a.cap_tokens) fail(LC_EINVAL, "lc_kv_upload_slot: n_tokens exceeds capacity");
        h->set_device();
        const Arena& a = h->a;
        ck(cudaMemcpy(h->kv_ptr(0, slot), keys, (size_t)n_tokens * a.d * h->kv_elem, cudaMemcpyHostToDevice), "K");
        ck(cudaMemcpy(h->kv_ptr(1, slot), values, (size_t)n_tokens * a.d * h->kv_elem, cudaMemcpyHostToDevice), "V");
        SlotState st;
        ck(cudaMemcpy(&st, a.state + slot, sizeof st, cudaMemcpyDeviceToHost), "state");
        st.n_tokens = n_tokens;
        ck(cudaMemcpy(a.state + slot, &st, sizeof st, cudaMemcpyHostToDevice), "state");
        h->hs[slot].n_tokens = n_tokens;
        ++h->version;
    });
}

int lc_kv_download_slot(lc_index_t h, uint32_t slot, void* keys, void* values, uint32_t n_tokens) {
    return guard([&] {
        if (!h || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_kv_download_slot: bad argument");
        sync_host(h);
        if (n_tokens > h->hs[slot].n_tokens) fail(LC_EINVAL, "lc_kv_download_slot: beyond the store");
        h->set_device();
        ck(cudaDeviceSynchronize(), "sync");
        const Arena& a = h->a;
        if (keys) ck(cudaMemcpy(keys, h->kv_ptr(0, slot), (size_t)n_tokens * a.d * h->kv_elem, cudaMemcpyDeviceToHost), "K");
        if (values) ck(cudaMemcpy(values, h->kv_ptr(1, slot), (size_t)n_tokens * a.d * h->kv_elem, cudaMemcpyDeviceToHost), "V");
    });
}

int lc_kv_append(lc_index_t h, const void* keys_dev, const void* values_dev, void* stream) {
    return guard([&] {
        if (!h || !keys_dev || !values_dev) fail(LC_EINVAL, "lc_kv_append: null argument");
        sync_host(h);
        h->set_device();
        for (auto& s : h->hs) {
            if (!s.loaded) fail(LC_EINVAL, "lc_kv_append: every slot must be uploaded or built");
            if (s.n_tokens >= h->a.cap_tokens) fail(LC_ENOMEM, "lc_kv_append: token capacity exhausted");
        }
        ck(launch_append(h->a, keys_dev, values_dev, (cudaStream_t)stream), "k_append");
        for (auto& s : h->hs) s.n_tokens += 1;
        ++h->version;
    });
}

static void validate_budgets(const lc_budgets* b) {
    if (!b) fail(LC_EINVAL, "null budgets");
    // Budgets::validate (retriever.cpp:11-17)
    if (b->unit_topk < 1) fail(LC_EINVAL, "unit_topk must be >= 1");
    if (b->mode == LC_MODE_FIXED_CLUSTER_COUNT && b->cluster_topk < 1) fail(LC_EINVAL, "cluster_topk must be >= 1");
    if (b->mode == LC_MODE_TOKEN_BUDGET && b->token_budget < 1) fail(LC_EINVAL, "token_budget must be >= 1");
    if (b->mode > 1) fail(LC_EINVAL, "unknown selection mode");
    if (b->unit_topk > 64) fail(LC_EINVAL, "unit_topk > 64 is not supported by the device kernel");
}

static void ensure_streams(lc_index_t h, uint32_t groups) {
    while (h->group_streams.size() < groups) {
        cudaStream_t s;
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
        h->group_streams.push_back(s);
    }
    while (h->group_events.size() < groups + 1) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
        h->group_events.push_back(e);
    }
}

static void retrieve_impl(lc_index_t h, const float* q_dev, const lc_budgets* b, uint32_t flags,
                          const uint32_t* buf_off, const uint32_t* buf_ids, float* out_dev,
                          cudaStream_t st, const float* q_in = nullptr, uint32_t first = 0,
                          uint32_t count = 0xffffffffu) {
    validate_budgets(b);
    if (!q_dev) fail(LC_EINVAL, "null q");
    if (flags > 2) fail(LC_EINVAL, "bad buffer flags");
    if (flags == LC_BUFFER_LIST && (!buf_off || !buf_ids)) fail(LC_EINVAL, "LC_BUFFER_LIST needs id lists");
    for (auto& s : h->hs)
        if (!s.loaded) fail(LC_EINVAL, "retrieve: every slot must be uploaded or built");
    h->set_device();
    Arena a = h->a;
    a.max_cand = (needed_candidates(h, std::min<uint32_t>(b->unit_topk, 64)) + 1) & ~1u;  // 8-byte key rows
    uint32_t pmax = 1;
    for (auto& s : h->hs) pmax = std::max(pmax, s.P);
    if (select3_pick_smem(a) > 200 * 1024) fail(LC_EINVAL, "retrieve: chunk capacity too large for k_pickq");
    const uint32_t max_union = needed_candidates(h, std::min<uint32_t>(a.G * std::min<uint32_t>(b->unit_topk, 64), 4096));
    const uint32_t kc8 = (a.max_cand + 7) & ~7u;  // k_select's per-head capacity
    // k_fine -> k_pickq: lo key, weight, hi per candidate; k_select's large-R path: key, list
    const size_t need = (size_t)a.n_slots * a.G * std::max<size_t>((size_t)a.max_cand * 20, (size_t)kc8 * 12);
    if (h->sel_scratch_bytes < need) {
        if (h->sel_scratch) cudaFree(h->sel_scratch);
        h->sel_scratch = nullptr;
        h->sel_scratch_bytes = 0;
        if (cudaMalloc(&h->sel_scratch, need) != cudaSuccess) {
            cudaGetLastError();
            fail(LC_ENOMEM, "selection scratch allocation failed");
        }
        h->sel_scratch_bytes = need;
    }
    // k_coarse -> k_fine -> k_pickq -> k_spans (selection, per slot group), then
    // one persistent k_attend over every slot (its grid barrier needs the whole GPU)
    uint32_t max_fanout = 0;
    for (auto& s : h->hs)
        for (uint32_t f : s.fanout) max_fanout = std::max(max_fanout, f);
    // streamed attention: the selection publishes each slot's tasks as it
    // finishes and the attention grid starts on them without waiting for the
    // slowest slot (one selection launch, one attention launch)
    const AttQueueDev* aq_use = nullptr;
    bool fused_ok = false;
    const uint32_t ncount = count == 0xffffffffu ? a.n_slots - std::min(first, a.n_slots) : count;
    if (out_dev && !a.kv_f32 && std::min<uint32_t>(h->desc.slot_groups, ncount) <= 1 &&
        !(getenv("LC_ATT_QUEUE") && atoi(getenv("LC_ATT_QUEUE")) == 0)) {
        if (!h->aq_mem) {
            const uint32_t cap = attend_queue_cap(a.d, a.G, a.n_slots);
            const size_t words = 8 + 2 * (size_t)a.n_slots + 4 * (size_t)cap;
            void* m = nullptr;
            if (cudaMalloc(&m, words * 4) != cudaSuccess) {
                cudaGetLastError();
                fail(LC_ENOMEM, "streamed attention queue allocation failed");
            }
            h->aq_mem = m;
            uint32_t* w = static_cast<uint32_t*>(m);
            h->aq.ctl = w;
            h->aq.sbase = w + 8;
            h->aq.scnt = h->aq.sbase + a.n_slots;
            h->aq.t_slot = h->aq.scnt + a.n_slots;
            h->aq.t_pos = h->aq.t_slot + cap;
            h->aq.t_cnt = h->aq.t_pos + cap;
            h->aq.tag = h->aq.t_cnt + cap;
            h->aq.cap = cap;
            ck(cudaMemset(w, 0, (8 + 2 * (size_t)a.n_slots + 3 * (size_t)cap) * 4), "queue init");
            ck(cudaMemset(h->aq.tag, 0xff, (size_t)cap * 4), "queue tags");
        }
        h->aq.n = ncount;
        // tasks of >= 512 tokens when the launch fills the GPU; few slots (one
        // layer of a layer-by-layer decode) cut finer so more warps share them
        h->aq.cmin = ncount >= 128 ? 512u : 128u;
        if (const char* ev = getenv("LC_ATT_QC")) h->aq.cmin = (uint32_t)std::max(16, atoi(ev)) & ~15u;  // experiments
        aq_use = &h->aq;
    }
    auto run_group = [&](Arena ag, uint32_t count, cudaStream_t gs, uint32_t gi) {
        // the fused per-slot kernel when the shape fits on chip, else the four-kernel chain
        const cudaError_t ef = launch_fused(ag, q_dev, q_in, b->unit_topk, b->mode, b->cluster_topk, b->token_budget,
                                            b->sink_size, flags, buf_off, buf_ids, h->sel_scratch, kc8, max_union,
                                            pmax, max_fanout, count, gs, aq_use);
        if (ef == cudaSuccess) {
            fused_ok = true;
            h->last_launches += 1;
            return;
        }
        if (ef != cudaErrorNotSupported) fail(LC_ECUDA, std::string("k_select: ") + cudaGetErrorString(ef));
        cudaGetLastError();
        const cudaError_t e = launch_select3(ag, q_dev, b->unit_topk, b->mode, b->cluster_topk, b->token_budget,
                                             b->sink_size, flags, buf_off, buf_ids, h->sel_scratch, a.max_cand,
                                             max_union, pmax, count, h->fine_ctr + 32 * gi,
                                             h->pick_ord + (size_t)16 * ag.G * ag.slot0, gs, q_in);
        if (e != cudaSuccess)
            fail(LC_ECUDA, std::string("k_select3: ") + g_select3_where + ": " + cudaGetErrorString(e));
        h->last_launches += 4;
    };
    h->last_launches = 0;
    if (count == 0xffffffffu) count = a.n_slots - std::min(first, a.n_slots);
    if (first >= a.n_slots || count == 0 || count > a.n_slots - first) fail(LC_EINVAL, "retrieve: bad slot range");
    const uint32_t groups = std::max<uint32_t>(1, std::min<uint32_t>(h->desc.slot_groups, count));

    if (groups == 1) {
        a.slot0 = first;
        run_group(a, count, st, 0);
    } else {
        // fork: each slot group's selection runs on its own stream
        ensure_streams(h, groups);
        ck(cudaEventRecord(h->group_events[0], st), "fork");
        for (uint32_t gi = 0; gi < groups; ++gi) {
            const uint32_t s0 = first + (uint32_t)((uint64_t)count * gi / groups);
            const uint32_t s1 = first + (uint32_t)((uint64_t)count * (gi + 1) / groups);
            if (s1 == s0) continue;
            cudaStream_t gs = h->group_streams[gi];
            ck(cudaStreamWaitEvent(gs, h->group_events[0], 0), "fork wait");
            Arena ag = a;
            ag.slot0 = s0;
            run_group(ag, s1 - s0, gs, gi);
            ck(cudaEventRecord(h->group_events[gi + 1], gs), "join record");
            ck(cudaStreamWaitEvent(st, h->group_events[gi + 1], 0), "join");
        }
    }
    a.slot0 = first;
    if (out_dev) {
        ck(launch_attend(a, q_dev, out_dev, h->att_part, count, st, h->pg.n ? &h->pg : nullptr,
                         fused_ok ? aq_use : nullptr),
           "k_attend");
        h->last_launches += a.kv_f32 ? 2 : (fused_ok && aq_use) ? 2 : 2 * ((count + kMaxAttendSlots - 1) / kMaxAttendSlots);
    }
    h->last_flags = flags;
    h->last_valid = 1;
}

int lc_retrieve(lc_index_t h, const float* q_dev, const lc_budgets* b, uint32_t flags,
                const uint32_t* buf_off_dev, const uint32_t* buf_ids_dev, float* out_dev, void* stream) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "null handle");
        retrieve_impl(h, q_dev, b, flags, buf_off_dev, buf_ids_dev, out_dev, (cudaStream_t)stream);
    });
}

int lc_retrieve_slots(lc_index_t h, uint32_t first_slot, uint32_t n_slots, const float* q_dev,
                      const lc_budgets* b, uint32_t flags, const uint32_t* buf_off_dev,
                      const uint32_t* buf_ids_dev, float* out_dev, void* stream) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "null handle");
        retrieve_impl(h, q_dev, b, flags, buf_off_dev, buf_ids_dev, out_dev, (cudaStream_t)stream, nullptr,
                      first_slot, n_slots);
    });
}

int lc_set_gather(lc_index_t h, uint32_t n_peers, const uint64_t* peer_out, const uint64_t* peer_flag,
                  const uint32_t* row_of_slot, uint64_t my_flag, uint32_t rows_per_wait) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "null handle");
        h->set_device();
        ck(cudaDeviceSynchronize(), "sync");
        if (h->pg_mem) cudaFree(h->pg_mem);
        h->pg_mem = nullptr;
        h->pg = PeerGather{nullptr, nullptr, nullptr, 0u};
        ++h->version;  // cached host-call graphs hold the old epilogue
        if (n_peers == 0) return;
        if (!peer_out || !peer_flag || !row_of_slot || !my_flag || rows_per_wait == 0)
            fail(LC_EINVAL, "lc_set_gather: null argument");
        const uint32_t S = h->a.n_slots;
        // one allocation: [n] out pointers, [n] flag pointers, [S] rows, wait count
        const size_t bytes = (size_t)n_peers * 16 + (size_t)S * 4 + 16;
        void* m = nullptr;
        if (cudaMalloc(&m, bytes) != cudaSuccess) {
            cudaGetLastError();
            fail(LC_ENOMEM, "lc_set_gather: allocation failed");
        }
        h->pg_mem = m;
        unsigned char* b = static_cast<unsigned char*>(m);
        ck(cudaMemcpy(b, peer_out, (size_t)n_peers * 8, cudaMemcpyHostToDevice), "peer out");
        ck(cudaMemcpy(b + (size_t)n_peers * 8, peer_flag, (size_t)n_peers * 8, cudaMemcpyHostToDevice), "peer flags");
        ck(cudaMemcpy(b + (size_t)n_peers * 16, row_of_slot, (size_t)S * 4, cudaMemcpyHostToDevice), "rows");
        h->pg_done = reinterpret_cast<unsigned int*>(b + (size_t)n_peers * 16 + (size_t)S * 4);
        ck(cudaMemset(h->pg_done, 0, 16), "wait count");
        h->pg = PeerGather{reinterpret_cast<float* const*>(b), reinterpret_cast<unsigned int* const*>(b + (size_t)n_peers * 8),
                           reinterpret_cast<const uint32_t*>(b + (size_t)n_peers * 16), n_peers};
        h->pg_myflag = reinterpret_cast<unsigned int*>(my_flag);
        h->pg_expect = rows_per_wait;
    });
}

int lc_gather_wait(lc_index_t h, void* stream) {
    return guard([&] {
        if (!h || !h->pg.n) fail(LC_EINVAL, "lc_gather_wait: no gather configured (lc_set_gather)");
        h->set_device();
        ck(launch_gather_wait(h->pg_myflag, h->pg_done, h->pg_expect, h->a.err, (cudaStream_t)stream),
           "k_gather_wait");
    });
}

int lc_sparse_attention(lc_index_t h, const float* q_dev, float* out_dev, void* stream) {
    return guard([&] {
        if (!h || !q_dev || !out_dev) fail(LC_EINVAL, "lc_sparse_attention: null argument");
        if (!h->last_valid) fail(LC_EINVAL, "lc_sparse_attention: no selection yet");
        h->set_device();
        Arena a = h->a;
        a.slot0 = 0;
        cudaEvent_t* ev = nullptr;
        if (h->att_ev_used * 2 + 2 <= h->att_ev.size()) ev = &h->att_ev[2 * h->att_ev_used++];
        ck(launch_attend(a, q_dev, out_dev, h->att_part, a.n_slots, (cudaStream_t)stream, nullptr, nullptr, ev),
           "k_attend");
    });
}

int lc_attend_timing(lc_index_t h, uint32_t n_launches, float* ms_sum, uint32_t* timed) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "lc_attend_timing: null handle");
        h->set_device();
        if (ms_sum || timed) {
            float sum = 0.f;
            uint32_t n = 0;
            if (!h->att_ev.empty()) ck(cudaEventSynchronize(h->att_ev[2 * (h->att_ev_used ? h->att_ev_used - 1 : 0) + 1]), "sync");
            for (size_t i = 0; i < h->att_ev_used; ++i) {
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, h->att_ev[2 * i], h->att_ev[2 * i + 1]) != cudaSuccess) continue;
                sum += ms;
                ++n;
            }
            if (ms_sum) *ms_sum = sum;
            if (timed) *timed = n;
        }
        for (cudaEvent_t e : h->att_ev) cudaEventDestroy(e);
        h->att_ev.clear();
        h->att_ev_used = 0;
        for (uint32_t i = 0; i < 2 * n_launches; ++i) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "event");
            h->att_ev.push_back(e);
        }
    });
}

static void graft_impl(lc_index_t h, const uint32_t* take, const uint32_t* kind, const uint32_t* level,
                       const float* reps_host, lc_graft_report* reports_dev, cudaStream_t st) {
    if (!take) fail(LC_EINVAL, "null take");
    sync_host(h);
    bool any = false;
    for (uint32_t s = 0; s < h->a.n_slots; ++s) {
        const HostSlot& hs = h->hs[s];
        if (!take[s]) continue;
        if (!hs.loaded) fail(LC_EINVAL, "graft: slot not loaded");
        if (take[s] > hs.n_tokens - hs.chunked_end) fail(LC_EINVAL, "graft: take exceeds the buffered tokens");
        if (hs.n_chunks >= h->a.cap_chunks) fail(LC_ENOMEM, "graft: chunk capacity exhausted");
        any = true;
    }
    if (!any) return;
    h->set_device();
    ck(cudaMemcpyAsync(h->take_dev, take, h->a.n_slots * 4, cudaMemcpyHostToDevice, st), "take H2D");
    if (reps_host)
        ck(cudaMemcpyAsync(h->reps_dev, reps_host, (size_t)h->a.n_slots * h->a.d * 4, cudaMemcpyHostToDevice, st),
           "reps H2D");
    ck(launch_graft(h->a, h->take_dev, h->desc.pooling, reports_dev ? (void*)reports_dev : (void*)h->rep_scratch,
                    reps_host ? h->reps_dev : nullptr, st),
       "k_graft");
    for (uint32_t s = 0; s < h->a.n_slots; ++s) {
        if (!take[s]) continue;
        HostSlot& hs = h->hs[s];
        hs.kind.push_back(kind ? kind[s] : 1u);
        hs.level.push_back(level ? level[s] : 0u);
        hs.chunked_end += take[s];
        hs.n_chunks += 1;
        ++h->version;
        if (!hs.rep.empty()) hs.rep.clear();  // prefill reps no longer complete
    }
    // take[] is a pageable host array: make the async copy complete before return
    ck(cudaStreamSynchronize(st), "graft sync");
}

int lc_graft(lc_index_t h, const uint32_t* take, const uint32_t* kind, const uint32_t* level,
             lc_graft_report* reports_dev, void* stream) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "null handle");
        graft_impl(h, take, kind, level, nullptr, reports_dev, (cudaStream_t)stream);
    });
}

// Every kCompactEvery decode steps, fold the slots' grafted chunks into the
// member CSR (k_compact; slots with >= kCompactMin grafts).  A fixed launch in
// the step sequence, so a captured run of steps carries it too.  Skipped when
// the chunk table does not fit the kernel's shared-memory staging (1M-token
// contexts): the selection then keeps scanning the grafted tail.
constexpr uint32_t kCompactEvery = 128, kCompactMin = 64;
static void maybe_compact(lc_index_t h, cudaStream_t st) {
    if (++h->steps_since_compact < kCompactEvery) return;
    h->steps_since_compact = 0;
    if (compact_smem(h->a) + 1024 > (size_t)dev_props().smem_blk) return;
    ck(launch_compact(h->a, kCompactMin, st), "k_compact");
}

int lc_decode_step(lc_index_t h, const float* q_dev, const void* keys_dev, const void* values_dev,
                   const lc_budgets* b, const uint32_t* take, const uint32_t* kind, const uint32_t* level,
                   float* out_dev, lc_graft_report* reports_dev, void* stream) {
    return guard([&] {
        if (!h || !keys_dev || !values_dev) fail(LC_EINVAL, "lc_decode_step: null argument");
        cudaStream_t st = (cudaStream_t)stream;
        sync_host(h);
        retrieve_impl(h, q_dev, b, LC_BUFFER_STREAM, nullptr, nullptr, out_dev, st);
        for (auto& s : h->hs)
            if (s.n_tokens >= h->a.cap_tokens) fail(LC_ENOMEM, "decode_step: token capacity exhausted");
        ck(launch_append(h->a, keys_dev, values_dev, st), "k_append");
        for (auto& s : h->hs) s.n_tokens += 1;
        ++h->version;
        if (take) graft_impl(h, take, kind, level, nullptr, reports_dev, st);
        maybe_compact(h, st);
    });
}

int lc_compact(lc_index_t h, uint32_t min_grafted, void* stream) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "null handle");
        h->set_device();
        if (compact_smem(h->a) + 1024 > (size_t)dev_props().smem_blk)
            fail(LC_EINVAL, "lc_compact: the chunk table is too large for the compaction kernel");
        ck(launch_compact(h->a, min_grafted, (cudaStream_t)stream), "k_compact");
        ++h->version;
    });
}

int lc_decode_step_async(lc_index_t h, const float* q_dev, const void* keys_dev, const void* values_dev,
                         const lc_budgets* b, const uint32_t* take_dev, const uint32_t* kind_dev,
                         const uint32_t* level_dev, float* out_dev, lc_graft_report* reports_dev, void* stream) {
    return guard([&] {
        if (!h || !keys_dev || !values_dev) fail(LC_EINVAL, "lc_decode_step_async: null argument");
        cudaStream_t st = (cudaStream_t)stream;
        // no host reads or writes of the stream cursors: every launch below takes
        // its slot state from the device, so the sequence is graph-capturable
        retrieve_impl(h, q_dev, b, LC_BUFFER_STREAM, nullptr, nullptr, out_dev, st);
        ck(launch_append(h->a, keys_dev, values_dev, st), "k_append");
        h->last_launches += 1;
        if (take_dev) {
            ck(launch_graft(h->a, take_dev, h->desc.pooling, reports_dev ? (void*)reports_dev : (void*)h->rep_scratch,
                            nullptr, st, kind_dev, level_dev),
               "k_graft");
            h->last_launches += 1;
        }
        maybe_compact(h, st);
        h->dev_ahead = true;
        ++h->version;
    });
}

int lc_graft_rep(lc_index_t h, const uint32_t* take, const uint32_t* kind, const uint32_t* level,
                 const float* reps_host, lc_graft_report* reports_dev, void* stream) {
    return guard([&] {
        if (!h || !reps_host) fail(LC_EINVAL, "lc_graft_rep: null argument");
        graft_impl(h, take, kind, level, reps_host, reports_dev, (cudaStream_t)stream);
    });
}

int lc_chunk_rep(lc_index_t h, uint32_t slot, uint32_t start, uint32_t take, float* rep_host) {
    return guard([&] {
        if (!h || !rep_host || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_chunk_rep: bad argument");
        sync_host(h);
        if (take == 0 || start + take > h->hs[slot].n_tokens) fail(LC_EINVAL, "lc_chunk_rep: rows outside the store");
        h->set_device();
        uint32_t err0 = 0;
        ck(cudaMemcpy(&err0, h->a.err, 4, cudaMemcpyDeviceToHost), "err");
        ck(launch_chunk_rep(h->a, slot, start, take, h->desc.pooling, h->reps_dev, 0), "k_chunk_rep");
        ck(cudaMemcpy(rep_host, h->reps_dev, (size_t)h->a.d * 4, cudaMemcpyDeviceToHost), "rep D2H");
        uint32_t err = 0;
        ck(cudaMemcpy(&err, h->a.err, 4, cudaMemcpyDeviceToHost), "err");
        if ((err & ~err0) & kErrZeroNorm) {
            ck(cudaMemcpy(h->a.err, &err0, 4, cudaMemcpyHostToDevice), "err restore");
            fail(LC_ERUNTIME, "chunk_representative: zero-norm pooled key");  // index.cpp:36-37
        }
    });
}

int lc_sparse_attention_ids(lc_index_t h, uint32_t slot, const float* q_dev, const uint32_t* ids_host,
                            uint32_t n_ids, float* out_dev, void* stream) {
    return guard([&] {
        if (!h || !q_dev || !out_dev || slot >= h->a.n_slots) fail(LC_EINVAL, "lc_sparse_attention_ids: bad argument");
        sync_host(h);
        if (n_ids == 0) fail(LC_EINVAL, "sparse_attention: empty active set");  // retriever.cpp:43
        if (!ids_host) fail(LC_EINVAL, "lc_sparse_attention_ids: null ids");
        const HostSlot& hs = h->hs[slot];
        if (n_ids > h->a.cap_tokens) fail(LC_EINVAL, "sparse_attention: more ids than the token capacity");
        const uint32_t all = (1u << h->a.G) - 1u;
        std::vector<uint32_t> rows(n_ids);
        for (uint32_t i = 0; i < n_ids; ++i) {
            if (ids_host[i] >= hs.n_tokens) fail(LC_EINVAL, "sparse_attention: token id out of range");
            rows[i] = ids_host[i] | (all << 24);
        }
        h->set_device();
        cudaStream_t st = (cudaStream_t)stream;
        Arena a = h->a;
        ck(cudaMemcpyAsync(a.rows + (size_t)slot * a.cap_tokens, rows.data(), (size_t)n_ids * 4, cudaMemcpyHostToDevice, st),
           "rows H2D");
        ck(cudaMemcpyAsync(a.slot_tok + slot, &n_ids, 4, cudaMemcpyHostToDevice, st), "count H2D");
        a.slot0 = slot;
        // the attention kernels address q / out as [slot][G][d] arrays: shift the
        // caller's [G][d] buffers so that row `slot` lands on them
        const size_t off = (size_t)slot * a.G * a.d;
        ck(launch_attend(a, q_dev - off, out_dev - off, h->att_part, 1, st), "k_attend");
        ck(cudaStreamSynchronize(st), "attention sync");  // host arrays above are pageable
        h->last_valid = 0;  // the slot's row list no longer matches its selection
    });
}

int lc_retrieve_host(lc_index_t h, const float* q_host, const lc_budgets* b, uint32_t flags,
                     float* out_host, void* stream) {
    return guard([&] {
        if (!h || !q_host || !out_host) fail(LC_EINVAL, "lc_retrieve_host: null argument");
        if (flags == LC_BUFFER_LIST) fail(LC_EINVAL, "lc_retrieve_host: LC_BUFFER_LIST needs device lists");
        h->set_device();
        cudaStream_t st = (cudaStream_t)stream;
        const size_t bytes = (size_t)h->a.n_slots * h->a.G * h->a.d * 4;
        validate_budgets(b);
        // the decode step's kernels replay as one CUDA graph on the handle's own
        // stream (captured once per budgets / flags / index version), ordered
        // after the caller's stream; the copies stay outside the graph because
        // the host buffers may change from call to call
        if (!h->host_stream) {
            ck(cudaStreamCreateWithFlags(&h->host_stream, cudaStreamNonBlocking), "stream create");
            ck(cudaEventCreateWithFlags(&h->host_event, cudaEventDisableTiming), "event create");
        }
        ck(cudaEventRecord(h->host_event, st), "order after caller");
        ck(cudaStreamWaitEvent(h->host_stream, h->host_event, 0), "order after caller");
        // page-locked, device-mapped host buffers (cudaHostAlloc / torch pin_memory):
        // k_coarse reads q straight from host memory and k_attend writes the
        // outputs straight into it, so no copy-engine transfer sits between the
        // call and the kernels; other host memory goes through the staging copies
        auto mapped = [](const void* ptr) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            return at.type == cudaMemoryTypeHost && at.devicePointer == ptr && !getenv("LC_HOST_STAGED");
        };
        const bool zc = mapped(q_host) && mapped(out_host);
        if (!zc) ck(cudaMemcpyAsync(h->q_stage, q_host, bytes, cudaMemcpyHostToDevice, h->host_stream), "q H2D");
        const float* q_in = zc ? q_host : nullptr;
        float* out_k = zc ? out_host : h->out_stage;
        const bool same = h->host_exec && h->host_version == h->version && h->host_flags == flags &&
                          std::memcmp(&h->host_budgets, b, sizeof *b) == 0 && h->host_q == q_in &&
                          h->host_out == out_k && h->host_scratch == h->sel_scratch;
        if (!same) {
            if (h->host_exec) cudaGraphExecDestroy(h->host_exec);
            h->host_exec = nullptr;
            // one eager run sizes every scratch buffer, then the capture
            retrieve_impl(h, h->q_stage, b, flags, nullptr, nullptr, out_k, h->host_stream, q_in);
            ck(cudaStreamSynchronize(h->host_stream), "warm-up");
            cudaGraph_t g = nullptr;
            ck(cudaStreamBeginCapture(h->host_stream, cudaStreamCaptureModeThreadLocal), "capture begin");
            try {
                retrieve_impl(h, h->q_stage, b, flags, nullptr, nullptr, out_k, h->host_stream, q_in);
            } catch (...) {
                cudaStreamEndCapture(h->host_stream, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            ck(cudaStreamEndCapture(h->host_stream, &g), "capture end");
            const cudaError_t e = cudaGraphInstantiate(&h->host_exec, g, 0);
            cudaGraphDestroy(g);
            ck(e, "graph instantiate");
            h->host_version = h->version;
            h->host_flags = flags;
            h->host_budgets = *b;
            h->host_q = q_in;
            h->host_out = out_k;
            h->host_scratch = h->sel_scratch;  // a later reallocation invalidates the graph
        }
        ck(cudaGraphLaunch(h->host_exec, h->host_stream), "graph launch");
        if (!zc) ck(cudaMemcpyAsync(out_host, h->out_stage, bytes, cudaMemcpyDeviceToHost, h->host_stream), "out D2H");
        ck(cudaStreamSynchronize(h->host_stream), "stream sync");
        h->last_flags = flags;
        h->last_valid = 1;
    });
}

int lc_selection_download(lc_index_t h, uint32_t slot, uint32_t g, lc_selection_info* info, uint32_t* units,
                          uint64_t units_cap, uint32_t* clusters, uint64_t clusters_cap, uint32_t* active,
                          uint64_t active_cap) {
    return guard([&] {
        if (!h || slot >= h->a.n_slots || g >= h->a.G) fail(LC_EINVAL, "lc_selection_download: bad argument");
        sync_host(h);
        if (!h->last_valid) fail(LC_EINVAL, "no selection yet");
        h->set_device();
        ck(cudaDeviceSynchronize(), "sync");
        const Arena& a = h->a;
        uint32_t err = 0;
        ck(cudaMemcpy(&err, a.err, 4, cudaMemcpyDeviceToHost), "err");
        QInfo qi;
        ck(cudaMemcpy(&qi, a.qinfo + (size_t)slot * a.G + g, sizeof qi, cudaMemcpyDeviceToHost), "qinfo");
        if (info) {
            info->n_units = qi.n_units;
            info->n_clusters = qi.n_clusters;
            info->degenerate = qi.degenerate;
            info->error = qi.error | err;
            info->scanned_centroids = qi.scanned;
            info->n_active = qi.n_active;
        }
        const HostSlot& hs = h->hs[slot];
        if (qi.degenerate) {
            if (units) for (uint64_t i = 0; i < std::min<uint64_t>(units_cap, hs.P); ++i) units[i] = (uint32_t)i;
            if (clusters) for (uint64_t i = 0; i < std::min<uint64_t>(clusters_cap, hs.L); ++i) clusters[i] = (uint32_t)i;
        } else {
            if (units && qi.n_units)
                ck(cudaMemcpy(units, a.sel_units + ((size_t)slot * a.G + g) * a.cap_units,
                              std::min<uint64_t>(units_cap, qi.n_units) * 4, cudaMemcpyDeviceToHost), "units");
            if (clusters && qi.n_clusters)
                ck(cudaMemcpy(clusters, a.sel_clusters + ((size_t)slot * a.G + g) * a.cap_clusters,
                              std::min<uint64_t>(clusters_cap, qi.n_clusters) * 4, cudaMemcpyDeviceToHost),
                   "clusters");
        }
        if (active) {
            uint32_t ns = 0;
            ck(cudaMemcpy(&ns, a.n_spans + slot, 4, cudaMemcpyDeviceToHost), "n_spans");
            std::vector<Span> sp(ns);
            if (ns) ck(cudaMemcpy(sp.data(), a.spans + (size_t)slot * a.cap_spans, ns * sizeof(Span), cudaMemcpyDeviceToHost), "spans");
            std::vector<uint32_t> ids;
            for (const Span& s : sp)
                if ((s.len_mask >> g) & 1u)
                    for (uint32_t t = 0; t < (s.len_mask >> 8); ++t) ids.push_back(s.start + t);
            std::sort(ids.begin(), ids.end());
            ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
            if (info) info->n_active = ids.size();
            std::memcpy(active, ids.data(), std::min<uint64_t>(active_cap, ids.size()) * 4);
        }
    });
}

// Page-locked staging of one head's selection (lc_selection_stage /
// lc_selection_read_staged): [0] error bits, [16] QInfo, [48] span count,
// [64] units [cap_units], clusters [cap_clusters], spans [cap_spans].
static size_t stage_units_off() { return 64; }
static size_t stage_clusters_off(const Arena& a) { return 64 + (size_t)a.cap_units * 4; }
static size_t stage_spans_off(const Arena& a) {
    return (stage_clusters_off(a) + (size_t)a.cap_clusters * 4 + 15) & ~(size_t)15;
}

// Active ids of head g from the slot's union spans (ascending, disjoint runs;
// sorted defensively if not), as the reference's collect_active returns them.
static uint64_t expand_active(const Span* sp, uint32_t ns, uint32_t g, uint32_t* active, uint64_t cap) {
    uint64_t k = 0;
    bool sorted = true;
    uint32_t last = 0;
    std::vector<uint32_t> ids;
    for (uint32_t i = 0; i < ns; ++i) {
        if (!((sp[i].len_mask >> g) & 1u)) continue;
        const uint32_t len = sp[i].len_mask >> 8;
        for (uint32_t t = 0; t < len; ++t) {
            const uint32_t id = sp[i].start + t;
            if (k && id <= last) sorted = false;
            last = id;
            ids.push_back(id);
            ++k;
        }
    }
    if (!sorted) {
        std::sort(ids.begin(), ids.end());
        ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    }
    if (active) std::memcpy(active, ids.data(), std::min<uint64_t>(cap, ids.size()) * 4);
    return ids.size();
}

int lc_selection_stage(lc_index_t h, uint32_t slot, uint32_t g, void* stream) {
    return guard([&] {
        if (!h || slot >= h->a.n_slots || g >= h->a.G) fail(LC_EINVAL, "lc_selection_stage: bad argument");
        if (!h->last_valid) fail(LC_EINVAL, "no selection yet");
        h->set_device();
        const Arena& a = h->a;
        const size_t need = stage_spans_off(a) + (size_t)a.cap_spans * sizeof(Span);
        if (h->sel_stage_bytes < need) {
            if (h->sel_stage) cudaFreeHost(h->sel_stage);
            h->sel_stage = nullptr;
            h->sel_stage_bytes = 0;
            ck(cudaHostAlloc(reinterpret_cast<void**>(&h->sel_stage), need, cudaHostAllocDefault), "stage alloc");
            h->sel_stage_bytes = need;
        }
        cudaStream_t st = (cudaStream_t)stream;
        unsigned char* b = h->sel_stage;
        const size_t q = (size_t)slot * a.G + g;
        ck(cudaMemcpyAsync(b, a.err, 4, cudaMemcpyDeviceToHost, st), "err");
        ck(cudaMemcpyAsync(b + 16, a.qinfo + q, sizeof(QInfo), cudaMemcpyDeviceToHost, st), "qinfo");
        ck(cudaMemcpyAsync(b + 48, a.n_spans + slot, 4, cudaMemcpyDeviceToHost, st), "n_spans");
        ck(cudaMemcpyAsync(b + stage_units_off(), a.sel_units + q * a.cap_units, (size_t)a.cap_units * 4,
                           cudaMemcpyDeviceToHost, st), "units");
        ck(cudaMemcpyAsync(b + stage_clusters_off(a), a.sel_clusters + q * a.cap_clusters, (size_t)a.cap_clusters * 4,
                           cudaMemcpyDeviceToHost, st), "clusters");
        ck(cudaMemcpyAsync(b + stage_spans_off(a), a.spans + (size_t)slot * a.cap_spans, (size_t)a.cap_spans * sizeof(Span),
                           cudaMemcpyDeviceToHost, st), "spans");
        h->stage_slot = slot;
        h->stage_g = g;
        h->stage_valid = true;
    });
}

int lc_selection_read_staged(lc_index_t h, lc_selection_info* info, uint32_t* units, uint64_t units_cap,
                             uint32_t* clusters, uint64_t clusters_cap, uint32_t* active, uint64_t active_cap) {
    return guard([&] {
        if (!h) fail(LC_EINVAL, "lc_selection_read_staged: null handle");
        if (!h->stage_valid) fail(LC_EINVAL, "lc_selection_read_staged: nothing staged");
        const Arena& a = h->a;
        const unsigned char* b = h->sel_stage;
        uint32_t err, ns;
        QInfo qi;
        std::memcpy(&err, b, 4);
        std::memcpy(&qi, b + 16, sizeof qi);
        std::memcpy(&ns, b + 48, 4);
        if (ns > a.cap_spans) fail(LC_ERUNTIME, "lc_selection_read_staged: span count over capacity");
        const HostSlot& hs = h->hs[h->stage_slot];
        if (info) {
            info->n_units = qi.n_units;
            info->n_clusters = qi.n_clusters;
            info->degenerate = qi.degenerate;
            info->error = qi.error | err;
            info->scanned_centroids = qi.scanned;
            info->n_active = qi.n_active;
        }
        if (qi.degenerate) {
            if (units) for (uint64_t i = 0; i < std::min<uint64_t>(units_cap, hs.P); ++i) units[i] = (uint32_t)i;
            if (clusters) for (uint64_t i = 0; i < std::min<uint64_t>(clusters_cap, hs.L); ++i) clusters[i] = (uint32_t)i;
        } else {
            if (units)
                std::memcpy(units, b + stage_units_off(),
                            std::min<uint64_t>({units_cap, qi.n_units, a.cap_units}) * 4);
            if (clusters)
                std::memcpy(clusters, b + stage_clusters_off(a),
                            std::min<uint64_t>({clusters_cap, qi.n_clusters, a.cap_clusters}) * 4);
        }
        if (active || info) {
            const uint64_t n = expand_active(reinterpret_cast<const Span*>(b + stage_spans_off(a)), ns, h->stage_g,
                                             active, active_cap);
            if (info) info->n_active = n;
        }
    });
}

int lc_step_bytes(lc_index_t h, uint64_t* out) {
    return guard([&] {
        if (!h || !out) fail(LC_EINVAL, "null argument");
        h->set_device();
        ck(cudaDeviceSynchronize(), "sync");
        std::vector<unsigned long long> sb((size_t)h->a.n_slots * 4);
        ck(cudaMemcpy(sb.data(), h->a.step_bytes, sb.size() * 8, cudaMemcpyDeviceToHost), "step bytes");
        out[0] = out[1] = out[2] = out[3] = 0;
        for (uint32_t s = 0; s < h->a.n_slots; ++s)
            for (int k = 0; k < 4; ++k) out[k] += sb[(size_t)s * 4 + k];
    });
}

int lc_launch_count(lc_index_t h, uint32_t* out) {
    return guard([&] {
        if (!h || !out) fail(LC_EINVAL, "null argument");
        *out = h->last_launches;
    });
}

int lc_device_error(lc_index_t h, uint32_t* out, int clear) {
    return guard([&] {
        if (!h || !out) fail(LC_EINVAL, "null argument");
        h->set_device();
        ck(cudaDeviceSynchronize(), "sync");
        ck(cudaMemcpy(out, h->a.err, 4, cudaMemcpyDeviceToHost), "err");
        if (clear) ck(cudaMemset(h->a.err, 0, 4), "clear err");
    });
}

}  // extern "C"
