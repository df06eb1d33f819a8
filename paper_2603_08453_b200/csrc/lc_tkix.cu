// TKIX <-> device.  The reference's binary index
// container, byte for byte:
//
//   index_to_bytes  serialize.cpp:88-125   magic "TKIX", version 1, dim, chunks
//                                          (span + rep_key), fine clusters,
//                                          coarse units, cluster_of_chunk,
//                                          IndexConfig
//   save_index      serialize.cpp:127-148  index_to_bytes + the embedded token
//                                          store (texts, fp32 keys, fp32 values)
//   load_index      serialize.cpp:150-220  the inverse, with the same
//                                          truncation / size checks
//
// The slot-level entry points download a slot's live index (every graft
// included) and encode it, or decode a file and upload it into a slot, so a
// reference-built (or device-built) index can be cached on disk and the
// post-graft state compared with the reference as the byte stream the
// reference itself uses as its determinism check (test_index.cpp:239-318).
// Host-only code: no kernel runs here beyond the upload / download copies.
#include "../../include/lychee_b200.h"
#include "lc_common.cuh"
#include "lc_engine.hpp"

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr uint32_t kMagic = 0x58494b54u;  // "TKIX" little-endian (serialize.cpp:13)
constexpr uint32_t kVersion = 1u;

struct Writer {
    std::vector<uint8_t> buf;
    void raw(const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        buf.insert(buf.end(), b, b + n);
    }
    void u32(uint32_t v) { raw(&v, 4); }
    void u64(uint64_t v) { raw(&v, 8); }
    void f64(double v) { raw(&v, 8); }
    void f32s(const float* p, uint64_t n) {
        u64(n);
        raw(p, n * 4);
    }
    void u32s(const uint32_t* p, uint64_t n) {
        u64(n);
        raw(p, n * 4);
    }
    void str(const char* p, uint64_t n) {
        u64(n);
        raw(p, n);
    }
};

struct Reader {
    const uint8_t* p;
    uint64_t n, pos = 0;
    Reader(const uint8_t* p_, uint64_t n_) : p(p_), n(n_) {}
    void raw(void* dst, uint64_t k) {
        if (k > n - pos) lcx::fail(LC_ERUNTIME, "index file truncated");  // serialize.cpp:80
        std::memcpy(dst, p + pos, k);
        pos += k;
    }
    uint32_t u32() {
        uint32_t v;
        raw(&v, 4);
        return v;
    }
    uint64_t u64() {
        uint64_t v;
        raw(&v, 8);
        return v;
    }
    double f64() {
        double v;
        raw(&v, 8);
        return v;
    }
    uint64_t count(uint64_t elem) {  // a length prefix that must fit the remaining bytes
        const uint64_t k = u64();
        if (elem && k > (n - pos) / elem) lcx::fail(LC_ERUNTIME, "index file truncated");
        return k;
    }
};

// One decoded index in owning vectors (the reference's numbering).
struct IndexBuf {
    uint32_t dim = 0;
    std::vector<uint32_t> span4, fine_parent, fmo{0}, fmem, cmo{0}, cmem, coc;
    std::vector<float> rep, fcent, ccent;
    std::vector<double> frad, crad;
    std::vector<uint64_t> ftok;
    lc_index_config cfg{};

    lc_host_index view() {
        lc_host_index ix{};
        ix.dim = dim;
        ix.n_chunks = (uint32_t)(span4.size() / 4);
        ix.n_clusters = (uint32_t)frad.size();
        ix.n_units = (uint32_t)crad.size();
        ix.chunk_span = span4.data();
        ix.chunk_rep = rep.data();
        ix.fine_centroid = fcent.data();
        ix.fine_radius = frad.data();
        ix.fine_token_count = ftok.data();
        ix.fine_parent = fine_parent.data();
        ix.fine_member_off = fmo.data();
        ix.fine_members = fmem.data();
        ix.coarse_centroid = ccent.data();
        ix.coarse_radius = crad.data();
        ix.coarse_member_off = cmo.data();
        ix.coarse_members = cmem.data();
        ix.cluster_of_chunk = coc.data();
        return ix;
    }
};

// index_to_bytes (serialize.cpp:88-125)
void encode(const lc_host_index& ix, const lc_index_config& cfg, Writer& w) {
    const uint32_t d = ix.dim;
    if (!ix.chunk_span || !ix.chunk_rep || !ix.fine_centroid || !ix.fine_radius || !ix.fine_token_count ||
        !ix.fine_parent || !ix.fine_member_off || !ix.fine_members || !ix.coarse_centroid || !ix.coarse_radius ||
        !ix.coarse_member_off || !ix.coarse_members || !ix.cluster_of_chunk)
        lcx::fail(LC_EINVAL, "index_to_bytes: every index array (chunk representatives included) is required");
    w.u32(kMagic);
    w.u32(kVersion);
    w.u64(d);
    w.u64(ix.n_chunks);
    for (uint32_t j = 0; j < ix.n_chunks; ++j) {
        for (int k = 0; k < 4; ++k) w.u32(ix.chunk_span[4 * (size_t)j + k]);
        w.f32s(ix.chunk_rep + (size_t)j * d, d);
    }
    w.u64(ix.n_clusters);
    for (uint32_t c = 0; c < ix.n_clusters; ++c) {
        w.f32s(ix.fine_centroid + (size_t)c * d, d);
        w.f64(ix.fine_radius[c]);
        const uint32_t b = ix.fine_member_off[c], e = ix.fine_member_off[c + 1];
        w.u32s(ix.fine_members + b, e - b);
        w.u64(ix.fine_token_count[c]);
        w.u32(ix.fine_parent[c]);
    }
    w.u64(ix.n_units);
    for (uint32_t u = 0; u < ix.n_units; ++u) {
        w.f32s(ix.coarse_centroid + (size_t)u * d, d);
        w.f64(ix.coarse_radius[u]);
        const uint32_t b = ix.coarse_member_off[u], e = ix.coarse_member_off[u + 1];
        w.u32s(ix.coarse_members + b, e - b);
    }
    w.u32s(ix.cluster_of_chunk, ix.n_chunks);
    w.f64(cfg.avg_chunks_per_cluster);
    w.u32(cfg.max_coarse_units);
    w.u32(cfg.kmeans_iters);
    w.u32(cfg.pooling);
    w.u64(cfg.seed);
    w.u32(cfg.elem_bytes);
}

// the index part of load_index (serialize.cpp:160-208)
void decode(Reader& r, IndexBuf& b) {
    if (r.u32() != kMagic) lcx::fail(LC_ERUNTIME, "not an index file");
    if (r.u32() != kVersion) lcx::fail(LC_ERUNTIME, "unsupported index version");
    const uint64_t d64 = r.u64();
    if (d64 == 0 || d64 > 4096) lcx::fail(LC_ERUNTIME, "index file: bad dimension");
    const uint32_t d = (uint32_t)d64;
    b.dim = d;
    auto vec_f32 = [&](std::vector<float>& out) {
        const uint64_t k = r.count(4);
        if (k != d) lcx::fail(LC_ERUNTIME, "index file: vector length differs from dim");
        const size_t o = out.size();
        out.resize(o + k);
        r.raw(out.data() + o, k * 4);
    };
    auto vec_u32 = [&](std::vector<uint32_t>& out) {
        const uint64_t k = r.count(4);
        const size_t o = out.size();
        out.resize(o + k);
        r.raw(out.data() + o, k * 4);
        return k;
    };
    const uint64_t m = r.count(16 + 8);
    b.span4.resize(m * 4);
    for (uint64_t j = 0; j < m; ++j) {
        for (int k = 0; k < 4; ++k) b.span4[4 * j + k] = r.u32();
        vec_f32(b.rep);
    }
    const uint64_t l = r.count(8 + 8 + 8 + 8 + 4);
    for (uint64_t c = 0; c < l; ++c) {
        vec_f32(b.fcent);
        b.frad.push_back(r.f64());
        vec_u32(b.fmem);
        b.fmo.push_back((uint32_t)b.fmem.size());
        b.ftok.push_back(r.u64());
        b.fine_parent.push_back(r.u32());
    }
    const uint64_t p = r.count(8 + 8 + 8);
    for (uint64_t u = 0; u < p; ++u) {
        vec_f32(b.ccent);
        b.crad.push_back(r.f64());
        vec_u32(b.cmem);
        b.cmo.push_back((uint32_t)b.cmem.size());
    }
    vec_u32(b.coc);
    b.cfg.avg_chunks_per_cluster = r.f64();
    b.cfg.max_coarse_units = r.u32();
    b.cfg.kmeans_iters = r.u32();
    b.cfg.pooling = r.u32();
    b.cfg.seed = r.u64();
    b.cfg.elem_bytes = r.u32();
    if (m > 0xffffffffull || l > 0xffffffffull || p > 0xffffffffull) lcx::fail(LC_ERUNTIME, "index file: too large");
}

void copy_out(IndexBuf& b, lc_host_index* out) {
    const lc_host_index v = b.view();
    auto cp = [](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) std::memcpy(dst, src, bytes);
    };
    out->dim = v.dim;
    out->n_chunks = v.n_chunks;
    out->n_clusters = v.n_clusters;
    out->n_units = v.n_units;
    cp(out->chunk_span, b.span4.data(), b.span4.size() * 4);
    cp(out->chunk_rep, b.rep.data(), b.rep.size() * 4);
    cp(out->fine_centroid, b.fcent.data(), b.fcent.size() * 4);
    cp(out->fine_radius, b.frad.data(), b.frad.size() * 8);
    cp(out->fine_token_count, b.ftok.data(), b.ftok.size() * 8);
    cp(out->fine_parent, b.fine_parent.data(), b.fine_parent.size() * 4);
    cp(out->fine_member_off, b.fmo.data(), b.fmo.size() * 4);
    cp(out->fine_members, b.fmem.data(), b.fmem.size() * 4);
    cp(out->coarse_centroid, b.ccent.data(), b.ccent.size() * 4);
    cp(out->coarse_radius, b.crad.data(), b.crad.size() * 8);
    cp(out->coarse_member_off, b.cmo.data(), b.cmo.size() * 4);
    cp(out->coarse_members, b.cmem.data(), b.cmem.size() * 4);
    cp(out->cluster_of_chunk, b.coc.data(), b.coc.size() * 4);
}

void dims_of(const IndexBuf& b, uint64_t* dims) {
    dims[0] = b.dim;
    dims[1] = b.span4.size() / 4;
    dims[2] = b.frad.size();
    dims[3] = b.crad.size();
    dims[4] = 0;
    dims[5] = b.fmem.size();
    dims[6] = b.cmem.size();
    dims[7] = 0;
}

// download slot -> owning buffers (lc_index_download_slot into IndexBuf)
void download(lc_index_t h, uint32_t slot, IndexBuf& b) {
    uint64_t dims[8];
    int rc = lc_index_slot_dims(h, slot, dims);
    if (rc != LC_OK) lcx::fail(rc, lc_last_error());
    const uint64_t d = dims[0], m = dims[1], l = dims[2], p = dims[3];
    b.dim = (uint32_t)d;
    b.span4.resize(m * 4);
    b.rep.resize(m * d);
    b.fcent.resize(l * d);
    b.frad.resize(l);
    b.ftok.resize(l);
    b.fine_parent.resize(l);
    b.fmo.resize(l + 1);
    b.fmem.resize(dims[5]);
    b.ccent.resize(p * d);
    b.crad.resize(p);
    b.cmo.resize(p + 1);
    b.cmem.resize(dims[6]);
    b.coc.resize(m);
    lc_host_index v = b.view();
    rc = lc_index_download_slot(h, slot, &v);
    if (rc != LC_OK) lcx::fail(rc, lc_last_error());
}

std::vector<uint8_t> read_file(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) lcx::fail(LC_ERUNTIME, std::string("cannot read ") + path);
    std::vector<uint8_t> buf;
    uint8_t tmp[1 << 16];
    size_t k;
    while ((k = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + k);
    std::fclose(f);
    return buf;
}

}  // namespace

extern "C" {

int lc_tkix_encode(const lc_host_index* ix, const lc_index_config* cfg, uint8_t* buf, uint64_t cap, uint64_t* size) {
    return lcx::guard([&] {
        if (!ix || !cfg || !size) lcx::fail(LC_EINVAL, "lc_tkix_encode: null argument");
        Writer w;
        encode(*ix, *cfg, w);
        *size = w.buf.size();
        if (buf) std::memcpy(buf, w.buf.data(), std::min<uint64_t>(cap, w.buf.size()));
    });
}

int lc_tkix_decode_dims(const uint8_t* buf, uint64_t size, uint64_t* dims) {
    return lcx::guard([&] {
        if (!buf || !dims) lcx::fail(LC_EINVAL, "lc_tkix_decode_dims: null argument");
        Reader r(buf, size);
        IndexBuf b;
        decode(r, b);
        dims_of(b, dims);
        dims[7] = r.pos;  // bytes of the index part (the token store of a file follows)
    });
}

int lc_tkix_decode(const uint8_t* buf, uint64_t size, lc_host_index* out, lc_index_config* cfg) {
    return lcx::guard([&] {
        if (!buf || !out) lcx::fail(LC_EINVAL, "lc_tkix_decode: null argument");
        Reader r(buf, size);
        IndexBuf b;
        decode(r, b);
        copy_out(b, out);
        if (cfg) *cfg = b.cfg;
    });
}

int lc_index_set_config(lc_index_t h, uint32_t slot, const lc_index_config* cfg) {
    return lcx::guard([&] {
        if (!h || !cfg || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_index_set_config: bad argument");
        sync_host(h);
        h->hs[slot].cfg = *cfg;
    });
}

int lc_index_get_config(lc_index_t h, uint32_t slot, lc_index_config* cfg) {
    return lcx::guard([&] {
        if (!h || !cfg || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_index_get_config: bad argument");
        sync_host(h);
        *cfg = h->hs[slot].cfg;
    });
}

int lc_index_to_bytes(lc_index_t h, uint32_t slot, uint8_t* buf, uint64_t cap, uint64_t* size) {
    return lcx::guard([&] {
        if (!h || !size || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_index_to_bytes: bad argument");
        sync_host(h);
        if (!h->hs[slot].loaded) lcx::fail(LC_EINVAL, "lc_index_to_bytes: slot not loaded");
        IndexBuf b;
        download(h, slot, b);
        Writer w;
        encode(b.view(), h->hs[slot].cfg, w);
        *size = w.buf.size();
        if (buf) std::memcpy(buf, w.buf.data(), std::min<uint64_t>(cap, w.buf.size()));
    });
}

int lc_index_save(lc_index_t h, uint32_t slot, const char* path, const char* text_buf, const uint64_t* text_offs) {
    return lcx::guard([&] {
        if (!h || !path || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_index_save: bad argument");
        sync_host(h);
        if (!h->hs[slot].loaded) lcx::fail(LC_EINVAL, "lc_index_save: slot not loaded");
        IndexBuf b;
        download(h, slot, b);
        Writer w;
        encode(b.view(), h->hs[slot].cfg, w);
        // the token store (serialize.cpp:136-146): texts, then fp32 keys and values
        const uint64_t n = h->hs[slot].n_tokens, d = h->a.d;
        w.u64(n);
        for (uint64_t i = 0; i < n; ++i) {
            if (text_buf && text_offs) w.str(text_buf + text_offs[i], text_offs[i + 1] - text_offs[i]);
            else w.str("", 0);
        }
        std::vector<float> kv[2];
        for (int which = 0; which < 2; ++which) {
            kv[which].resize(n * d);
            if (h->a.kv_f32) {
                int rc = lc_kv_download_slot(h, slot, which ? nullptr : kv[0].data(), which ? kv[1].data() : nullptr,
                                             (uint32_t)n);
                if (rc != LC_OK) lcx::fail(rc, lc_last_error());
            } else {  // bf16 store: widen exactly (the values the device attends over)
                std::vector<uint16_t> raw(n * d);
                int rc = lc_kv_download_slot(h, slot, which ? nullptr : raw.data(), which ? raw.data() : nullptr,
                                             (uint32_t)n);
                if (rc != LC_OK) lcx::fail(rc, lc_last_error());
                for (size_t i = 0; i < raw.size(); ++i) {
                    const uint32_t bits = (uint32_t)raw[i] << 16;
                    std::memcpy(&kv[which][i], &bits, 4);
                }
            }
        }
        w.f32s(kv[0].data(), kv[0].size());
        w.f32s(kv[1].data(), kv[1].size());
        FILE* f = std::fopen(path, "wb");
        if (!f) lcx::fail(LC_ERUNTIME, std::string("cannot write ") + path);
        const size_t wrote = std::fwrite(w.buf.data(), 1, w.buf.size(), f);
        const int cl = std::fclose(f);
        if (wrote != w.buf.size() || cl != 0) lcx::fail(LC_ERUNTIME, std::string("short write to ") + path);
    });
}

int lc_index_load(lc_index_t h, uint32_t slot, const char* path, char* text_buf, uint64_t text_cap,
                  uint64_t* text_offs, uint64_t offs_cap, uint64_t* n_tokens) {
    return lcx::guard([&] {
        if (!h || !path || slot >= h->a.n_slots) lcx::fail(LC_EINVAL, "lc_index_load: bad argument");
        sync_host(h);
        const std::vector<uint8_t> file = read_file(path);
        Reader r(file.data(), file.size());
        IndexBuf b;
        decode(r, b);
        if (b.dim != h->a.d) lcx::fail(LC_EINVAL, "lc_index_load: index dimension differs from the engine's");
        const uint64_t n = r.count(8);
        uint64_t tpos = 0;
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t k = r.count(1);
            if (text_offs && i < offs_cap) text_offs[i] = tpos;
            if (text_buf && tpos + k <= text_cap) std::memcpy(text_buf + tpos, file.data() + r.pos, k);
            r.pos += k;
            tpos += k;
        }
        if (text_offs && n < offs_cap) text_offs[n] = tpos;
        const uint64_t d = b.dim;
        std::vector<float> kv[2];
        for (int which = 0; which < 2; ++which) {
            const uint64_t k = r.count(4);
            if (k != n * d) lcx::fail(LC_ERUNTIME, "index file: token store size mismatch");  // serialize.cpp:209-210
            kv[which].resize(k);
            r.raw(kv[which].data(), k * 4);
        }
        if (n > h->a.cap_tokens) lcx::fail(LC_EINVAL, "lc_index_load: token store exceeds the slot capacity");
        lc_host_index v = b.view();
        int rc;
        if (h->a.kv_f32) {
            rc = lc_index_upload_slot(h, slot, &v, kv[0].data(), kv[1].data(), (uint32_t)n);
        } else {  // the bf16 serving store rounds to nearest even, as lc_kv_append does
            std::vector<__nv_bfloat16> kb(n * d), vb(n * d);
            for (size_t i = 0; i < kb.size(); ++i) {
                kb[i] = __float2bfloat16_rn(kv[0][i]);
                vb[i] = __float2bfloat16_rn(kv[1][i]);
            }
            rc = lc_index_upload_slot(h, slot, &v, kb.data(), vb.data(), (uint32_t)n);
        }
        if (rc != LC_OK) lcx::fail(rc, lc_last_error());
        h->hs[slot].cfg = b.cfg;
        if (n_tokens) *n_tokens = n;
    });
}

}  // extern "C"
