/* ORACLE / TEST INFRASTRUCTURE ONLY -- see lc_oracle.h.
 *
 * Plain-C restatement of the reference's decode-step path.  Each function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/src).  Compiled with -ffp-contract=off so that every
 * fp64 product is rounded before it is added, as in the reference objects. */
#include "lc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* kernels.cpp:13-17 -- fp64, sequential j, float*float is exact in fp64 */
double lco_dot(const float* a, const float* b, size_t d) {
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) s += (double)a[i] * (double)b[i];
    return s;
}

/* kernels.cpp:19-23 */
double lco_l2_norm(const float* a, size_t d) {
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) s += (double)a[i] * (double)a[i];
    return sqrt(s);
}

/* kernels.cpp:25-32 -- diff in fp64, diff*diff rounded, then added */
double lco_l2_dist(const float* a, const float* b, size_t d) {
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) {
        double diff = (double)a[i] - (double)b[i];
        s += diff * diff;
    }
    return sqrt(s);
}

/* kernels.cpp:155-159 -- UB_i = dot(q, c_i) + qnorm * r_i */
void lco_upper_bounds(const float* q, const float* centroids, const double* radii, size_t n,
                      size_t d, double qnorm, double* scores) {
    for (size_t i = 0; i < n; ++i) scores[i] = lco_dot(q, centroids + i * d, d) + qnorm * radii[i];
}

typedef struct {
    uint32_t id;
    double s;
} scored;

/* retriever.cpp:31-34: score desc, then id asc */
static int cmp_scored(const void* pa, const void* pb) {
    const scored* a = (const scored*)pa;
    const scored* b = (const scored*)pb;
    if (a->s != b->s) return a->s > b->s ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

/* retriever.cpp:27-39 */
int lco_select_topk(const uint32_t* ids, const double* scores, size_t n, size_t k,
                    uint32_t* out, size_t* n_out) {
    if (k < 1) return 1;
    scored* s = (scored*)malloc(sizeof(scored) * (n ? n : 1));
    for (size_t i = 0; i < n; ++i) {
        s[i].id = ids[i];
        s[i].s = scores[i];
    }
    qsort(s, n, sizeof(scored), cmp_scored);
    size_t m = n < k ? n : k;
    for (size_t i = 0; i < m; ++i) out[i] = s[i].id;
    *n_out = m;
    free(s);
    return 0;
}

/* kernels.cpp:108-144 (attention_weights + attention_output, serial order) */
int lco_attention(const float* q, const float* keys, const float* values, const uint32_t* ids,
                  size_t n, size_t d, float* out) {
    if (n == 0) return 1; /* retriever.cpp:43 */
    double* w = (double*)malloc(sizeof(double) * n);
    const double scale = 1.0 / sqrt((double)d);
    for (size_t i = 0; i < n; ++i) w[i] = lco_dot(q, keys + (size_t)ids[i] * d, d) * scale;
    double m = -INFINITY;
    for (size_t i = 0; i < n; ++i) m = w[i] > m ? w[i] : m; /* std::max(m, w) */
    double z = 0.0;
    for (size_t i = 0; i < n; ++i) {
        w[i] = exp(w[i] - m);
        z += w[i];
    }
    const double inv_z = 1.0 / z;
    for (size_t i = 0; i < n; ++i) w[i] *= inv_z;
    for (size_t j = 0; j < d; ++j) {
        double acc = 0.0;
        for (size_t i = 0; i < n; ++i) acc += w[i] * (double)values[(size_t)ids[i] * d + j];
        out[j] = (float)acc;
    }
    free(w);
    return 0;
}

/* index.cpp:20-41 */
int lco_chunk_representative(const float* keys, size_t rows, size_t d, int max_pool,
                             float* out) {
    if (d == 0 || rows == 0) return 1;
    double* acc = (double*)calloc(d, sizeof(double));
    if (!max_pool) {
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < d; ++j) acc[j] += (double)keys[i * d + j];
        for (size_t j = 0; j < d; ++j) acc[j] /= (double)rows;
    } else {
        for (size_t j = 0; j < d; ++j) acc[j] = keys[j];
        for (size_t i = 1; i < rows; ++i)
            for (size_t j = 0; j < d; ++j) {
                double v = keys[i * d + j];
                acc[j] = acc[j] < v ? v : acc[j]; /* std::max(acc, v) */
            }
    }
    double n2 = 0.0; /* std::inner_product: init = init + a*b, sequential */
    for (size_t j = 0; j < d; ++j) n2 = n2 + acc[j] * acc[j];
    double norm = sqrt(n2);
    if (norm == 0.0) {
        free(acc);
        return 2; /* runtime_error: pooled key has zero norm */
    }
    for (size_t j = 0; j < d; ++j) out[j] = (float)(acc[j] / norm);
    free(acc);
    return 0;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* retriever.cpp:60-74 -- sink U chunk spans of the clusters U buffer, sort+unique */
static size_t collect_active(const lco_index* ix, const uint8_t* selected, uint32_t sink,
                             const uint32_t* buffer, size_t n_buffer, uint32_t* out) {
    size_t k = 0;
    const uint32_t n = ix->n_tokens;
    const uint32_t s = sink < n ? sink : n;
    for (uint32_t i = 0; i < s; ++i) out[k++] = i;
    for (uint32_t j = 0; j < ix->n_chunks; ++j)
        if (selected[ix->cluster_of_chunk[j]])
            for (uint32_t t = ix->chunk_start[j]; t < ix->chunk_end[j]; ++t) out[k++] = t;
    for (size_t i = 0; i < n_buffer; ++i) out[k++] = buffer[i];
    qsort(out, k, sizeof(uint32_t), cmp_u32);
    size_t u = 0;
    for (size_t i = 0; i < k; ++i)
        if (u == 0 || out[u - 1] != out[i]) out[u++] = out[i];
    return u;
}

/* retriever.cpp:78-167 */
int lco_retrieve(const lco_index* ix, const float* q, const lco_budgets* b,
                 const uint32_t* buffer, size_t n_buffer, int with_output, lco_result* res) {
    /* Budgets::validate (retriever.cpp:11-17) */
    if (b->unit_topk < 1) return 1;
    if (b->mode == 0 && b->cluster_topk < 1) return 1;
    if (b->mode == 1 && b->token_budget < 1) return 1;
    const size_t d = ix->d;
    res->scanned = 0;
    res->degenerate = 0;
    const uint64_t total = ix->n_tokens;
    const int fits = b->mode == 1 && total <= b->token_budget;
    uint8_t* sel = (uint8_t*)calloc(ix->L ? ix->L : 1, 1);
    if (fits || ix->n_chunks == 0) { /* retriever.cpp:86-95 */
        res->degenerate = 1;
        for (uint32_t u = 0; u < ix->P; ++u) res->units[u] = u;
        res->n_units = ix->P;
        for (uint32_t c = 0; c < ix->L; ++c) res->clusters[c] = c;
        res->n_clusters = ix->L;
        for (uint32_t t = 0; t < ix->n_tokens; ++t) res->active[t] = t;
        res->n_active = ix->n_tokens;
    } else {
        const double qnorm = lco_l2_norm(q, d);
        /* tier 1 (retriever.cpp:100-116) */
        double* us = (double*)malloc(sizeof(double) * ix->P);
        uint32_t* uid = (uint32_t*)malloc(sizeof(uint32_t) * ix->P);
        lco_upper_bounds(q, ix->coarse_centroid, ix->coarse_radius, ix->P, d, qnorm, us);
        res->scanned += ix->P;
        for (uint32_t u = 0; u < ix->P; ++u) uid[u] = u;
        size_t nu = 0;
        lco_select_topk(uid, us, ix->P, b->unit_topk, res->units, &nu);
        res->n_units = nu;
        /* tier 2 (retriever.cpp:118-138) */
        size_t nc = 0;
        for (size_t i = 0; i < nu; ++i) {
            uint32_t u = res->units[i];
            nc += ix->coarse_member_off[u + 1] - ix->coarse_member_off[u];
        }
        uint32_t* cand = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
        double* cs = (double*)malloc(sizeof(double) * (nc ? nc : 1));
        size_t k = 0;
        for (size_t i = 0; i < nu; ++i) {
            uint32_t u = res->units[i];
            for (uint32_t m = ix->coarse_member_off[u]; m < ix->coarse_member_off[u + 1]; ++m)
                cand[k++] = ix->coarse_members[m];
        }
        for (size_t i = 0; i < nc; ++i) {
            uint32_t c = cand[i];
            cs[i] = lco_dot(q, ix->fine_centroid + (size_t)c * d, d) + qnorm * ix->fine_radius[c];
        }
        res->scanned += nc;
        int rc = 0;
        if (b->mode == 0) { /* retriever.cpp:140-141 */
            size_t nsel = 0;
            rc = lco_select_topk(cand, cs, nc, b->cluster_topk, res->clusters, &nsel);
            res->n_clusters = nsel;
        } else { /* retriever.cpp:142-154: prefix fill, break at first overflow */
            uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
            size_t no = 0;
            rc = lco_select_topk(cand, cs, nc, nc, order, &no);
            uint64_t used = 0;
            size_t nsel = 0;
            for (size_t i = 0; i < no; ++i) {
                uint64_t t = ix->fine_token_count[order[i]];
                if (nsel > 0 && used + t > b->token_budget) break;
                res->clusters[nsel++] = order[i];
                used += t;
            }
            res->n_clusters = nsel;
            free(order);
        }
        for (size_t i = 0; i < res->n_clusters; ++i) sel[res->clusters[i]] = 1;
        res->n_active = collect_active(ix, sel, b->sink_size, buffer, n_buffer, res->active);
        free(us);
        free(uid);
        free(cand);
        free(cs);
        if (rc) {
            free(sel);
            return rc;
        }
    }
    free(sel);
    if (with_output && res->output)
        return lco_attention(q, ix->keys, ix->values, res->active, res->n_active, d, res->output);
    return 0;
}

/* ---- chunker (chunker.cpp:16-149), over arbitrary strings ---------------- */
static const char* const kSep[4][7] = {
    {"\n\n", "---", "***", "```", "}", "]", ">"},
    {".", "?", "!", "\xe3\x80\x82", "\xef\xbc\x9f", "\xef\xbc\x81", "\n"},
    {",", ";", ":", "\xef\xbc\x8c", "\xef\xbc\x9b", "\xef\xbc\x9a", "\xe3\x80\x81"},
    {" ", "\t", 0, 0, 0, 0, 0}};

static int ends_with(const char* s, size_t n, const char* suf) {
    size_t m = strlen(suf);
    return n >= m && memcmp(s + n - m, suf, m) == 0;
}

static size_t codepoints(const char* s) {
    size_t n = 0;
    for (; *s; ++s)
        if (((unsigned char)*s & 0xC0) != 0x80) ++n;
    return n;
}

static int is_strip(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

/* chunker.cpp:65-81; returns level or 0 for none */
static int classify_impl(const char* text, size_t n, int multichar_only) {
    if (n == 0) return 0;
    size_t ns = n;
    while (ns > 0 && is_strip(text[ns - 1])) --ns;
    for (int lv = 1; lv <= 4; ++lv) {
        if (lv <= 3) {
            for (int i = 0; i < 7 && kSep[lv - 1][i]; ++i) {
                const char* sep = kSep[lv - 1][i];
                if (multichar_only && codepoints(sep) < 2) continue;
                if (ends_with(text, n, sep) || ends_with(text, ns, sep)) return lv;
            }
        } else if (!multichar_only) {
            char last = text[n - 1];
            if (last == ' ' || last == '\t') return lv;
        }
    }
    return 0;
}

/* chunker.cpp:90-101 */
static int classify_pair(const char* prev, const char* text) {
    size_t np = strlen(prev), nt = strlen(text);
    int own = classify_impl(text, nt, 0);
    if (own == 1) return own;
    if (nt && np) {
        char* cat = (char*)malloc(np + nt + 1);
        memcpy(cat, prev, np);
        memcpy(cat + np, text, nt + 1);
        int sp = classify_impl(cat, np + nt, 1);
        free(cat);
        if (sp && (!own || sp < own)) return sp;
    }
    return own;
}

/* chunker.cpp:103-149 with min_len 8, max_len 16 */
static size_t segment_texts(const char* const* texts, size_t n, uint32_t* spans4) {
    const size_t min_len = 8, max_len = 16;
    size_t start = 0, k = 0;
    while (start < n) {
        size_t remaining = n - start;
        if (remaining < min_len) {
            spans4[4 * k] = (uint32_t)start; spans4[4 * k + 1] = (uint32_t)n;
            spans4[4 * k + 2] = 2; spans4[4 * k + 3] = 0; ++k;
            break;
        }
        size_t hi = remaining < max_len ? remaining : max_len;
        int best_level = 0;
        size_t best_len = 0;
        for (size_t len = min_len; len <= hi; ++len) {
            size_t pos = start + len - 1;
            const char* prev = pos > 0 ? texts[pos - 1] : "";
            int level = classify_pair(prev, texts[pos]);
            if (level && (best_level == 0 || level <= best_level)) {
                best_level = level;
                best_len = len;
            }
        }
        if (best_len > 0) {
            spans4[4 * k] = (uint32_t)start; spans4[4 * k + 1] = (uint32_t)(start + best_len);
            spans4[4 * k + 2] = 0; spans4[4 * k + 3] = (uint32_t)best_level; ++k;
            start += best_len;
        } else if (remaining >= max_len) {
            spans4[4 * k] = (uint32_t)start; spans4[4 * k + 1] = (uint32_t)(start + max_len);
            spans4[4 * k + 2] = 1; spans4[4 * k + 3] = 0; ++k;
            start += max_len;
        } else {
            spans4[4 * k] = (uint32_t)start; spans4[4 * k + 1] = (uint32_t)n;
            spans4[4 * k + 2] = 2; spans4[4 * k + 3] = 0; ++k;
            break;
        }
    }
    return k;
}

static const char* code_text(uint8_t c) { return c == 1 ? "\n" : (c == 2 ? "}" : ""); }

size_t lco_segment_codes(const uint8_t* codes, size_t n, uint32_t* spans4) {
    const char** t = (const char**)malloc(sizeof(char*) * (n ? n : 1));
    for (size_t i = 0; i < n; ++i) t[i] = code_text(codes[i]);
    size_t k = segment_texts(t, n, spans4);
    free(t);
    return k;
}

/* ---- streaming (streamer.cpp:29-165) ------------------------------------- */

/* flush_buffer (streamer.cpp:29-54) */
static int flush_buffer(lco_index* ix, uint32_t* span4, float* rep) {
    const uint32_t len = ix->n_tokens - ix->chunked_end;
    uint32_t take = 16, kind = 1, level = 0;
    if (ix->structure_aware) {
        uint32_t* sp = (uint32_t*)malloc(sizeof(uint32_t) * 4 * (len + 1));
        lco_segment_codes(ix->text_code + ix->chunked_end, len, sp);
        if (sp[2] != 2) { /* head span is not a tail */
            take = sp[1] - sp[0];
            kind = sp[2];
            level = sp[3];
        }
        free(sp);
    }
    span4[0] = ix->chunked_end;
    span4[1] = ix->chunked_end + take;
    span4[2] = kind;
    span4[3] = level;
    int rc = lco_chunk_representative(ix->keys + (size_t)ix->chunked_end * ix->d, take, ix->d, 0,
                                      rep);
    ix->chunked_end += take;
    return rc;
}

/* push_token (streamer.cpp:56-66); TokenStore::append id check (types.hpp:34-43) */
int lco_push_token(lco_index* ix, const float* key, const float* value, uint8_t code,
                   int* emitted, uint32_t* span4, float* rep) {
    if (ix->n_tokens >= ix->cap_tokens) return 2;
    const size_t d = ix->d;
    memcpy(ix->keys + (size_t)ix->n_tokens * d, key, d * sizeof(float));
    memcpy(ix->values + (size_t)ix->n_tokens * d, value, d * sizeof(float));
    ix->text_code[ix->n_tokens] = code;
    ix->n_tokens += 1;
    *emitted = 0;
    if (ix->n_tokens - ix->chunked_end >= 16) {
        *emitted = 1;
        return flush_buffer(ix, span4, rep);
    }
    return 0;
}

/* graft_chunk (streamer.cpp:68-143) */
int lco_graft_chunk(lco_index* ix, const uint32_t* span4, const float* rep,
                    lco_graft_report* out) {
    if (ix->L == 0) return 1;
    if (ix->n_chunks >= ix->cap_chunks) return 2;
    const size_t d = ix->d;
    uint64_t comps = 0;
    uint32_t best_cluster = 0;
    double best = -INFINITY;
    int scoped = !ix->graft_full;
    uint32_t lo = 0, hi = 0;
    if (scoped) {
        uint32_t best_unit = 0;
        double bus = -INFINITY;
        for (uint32_t u = 0; u < ix->P; ++u) {
            double s = lco_dot(rep, ix->coarse_centroid + (size_t)u * d, d);
            ++comps;
            if (s > bus) {
                bus = s;
                best_unit = u;
            }
        }
        lo = ix->coarse_member_off[best_unit];
        hi = ix->coarse_member_off[best_unit + 1];
        if (lo == hi) scoped = 0;
    }
    if (scoped) {
        for (uint32_t m = lo; m < hi; ++m) {
            uint32_t c = ix->coarse_members[m];
            double s = lco_dot(rep, ix->fine_centroid + (size_t)c * d, d);
            ++comps;
            if (s > best) {
                best = s;
                best_cluster = c;
            }
        }
    } else {
        comps = 0;
        for (uint32_t c = 0; c < ix->L; ++c) {
            double s = lco_dot(rep, ix->fine_centroid + (size_t)c * d, d);
            ++comps;
            if (s > best) {
                best = s;
                best_cluster = c;
            }
        }
    }
    float* mu = ix->fine_centroid + (size_t)best_cluster * d;
    const double n = (double)ix->fine_member_count[best_cluster];
    double* moved = (double*)malloc(sizeof(double) * d);
    float* nc = (float*)malloc(sizeof(float) * d);
    double norm2 = 0.0;
    for (size_t j = 0; j < d; ++j) {
        moved[j] = n * (double)mu[j] + (double)rep[j];
        norm2 += moved[j] * moved[j];
    }
    const double norm = sqrt(norm2);
    memcpy(nc, mu, sizeof(float) * d);
    if (norm > 0.0)
        for (size_t j = 0; j < d; ++j) nc[j] = (float)(moved[j] / norm);
    const double delta = lco_l2_dist(nc, mu, d);
    const double to_new = lco_l2_dist(rep, nc, d);
    memcpy(mu, nc, sizeof(float) * d);
    double r = ix->fine_radius[best_cluster] + delta;
    ix->fine_radius[best_cluster] = r > to_new ? r : to_new; /* std::max(r+delta, to_new) */
    ix->fine_token_count[best_cluster] += span4[1] - span4[0];
    const uint32_t unit = ix->fine_parent[best_cluster];
    const double dg = lco_l2_dist(rep, ix->coarse_centroid + (size_t)unit * d, d);
    if (ix->coarse_radius[unit] < dg) ix->coarse_radius[unit] = dg;
    const uint32_t cid = ix->n_chunks;
    ix->chunk_start[cid] = span4[0];
    ix->chunk_end[cid] = span4[1];
    ix->chunk_kind[cid] = span4[2];
    ix->chunk_level[cid] = span4[3];
    memcpy(ix->chunk_rep + (size_t)cid * d, rep, sizeof(float) * d);
    ix->cluster_of_chunk[cid] = best_cluster;
    ix->fine_member_count[best_cluster] += 1;
    ix->n_chunks += 1;
    out->chunk_id = cid;
    out->cluster_id = best_cluster;
    out->unit_id = unit;
    out->centroid_delta = delta;
    out->fine_radius = ix->fine_radius[best_cluster];
    out->coarse_radius = ix->coarse_radius[unit];
    out->distance_comps = comps;
    free(moved);
    free(nc);
    return 0;
}

/* decode_step (streamer.cpp:145-165): buffer ids before the push, retrieve +
 * attend, then push the step's token and graft any emitted chunk. */
int lco_decode_step(lco_index* ix, const float* q, const float* key, const float* value,
                    uint8_t code, const lco_budgets* b, lco_result* res, int* grafted,
                    lco_graft_report* out) {
    const uint32_t nb = ix->n_tokens - ix->chunked_end;
    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (nb ? nb : 1));
    for (uint32_t i = 0; i < nb; ++i) buf[i] = ix->chunked_end + i;
    int rc = lco_retrieve(ix, q, b, buf, nb, 1, res);
    free(buf);
    if (rc) return rc;
    int emitted = 0;
    uint32_t span4[4];
    float* rep = (float*)malloc(sizeof(float) * ix->d);
    rc = lco_push_token(ix, key, value, code, &emitted, span4, rep);
    *grafted = 0;
    if (!rc && emitted) {
        rc = lco_graft_chunk(ix, span4, rep, out);
        *grafted = rc == 0;
    }
    free(rep);
    return rc;
}

uint64_t lco_fnv1a64(const uint8_t* buf, size_t n) {
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= buf[i];
        h *= 1099511628211ull;
    }
    return h;
}
