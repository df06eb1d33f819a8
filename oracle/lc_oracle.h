/* ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * Plain-C restatement of the reference's per-decode-step path
 * (/root/reference/proj/src/{kernels,retriever,streamer,index,chunker}.cpp),
 * used by tests/ as an independent CPU checker next to the reference library
 * itself (oracle/_ref).  Parity is pinned: tests/test_oracle.py checks this
 * restatement bit-for-bit against oracle/_ref and the committed golden vectors
 * in tests/golden/.
 *
 * Numeric rules (same as the reference objects, which are compiled for
 * baseline x86-64 without FMA): every fp64 reduction is sequential in index
 * order, products are rounded before the add (-ffp-contract=off).
 */
#ifndef LC_ORACLE_H
#define LC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mutable SoA restatement of tierkv::HierarchicalIndex (index.hpp:25-73) plus
 * the TokenStore (types.hpp:25-57) and StreamState cursor (streamer.hpp:80-85).
 * Cluster membership is carried by cluster_of_chunk: the members of fine
 * cluster c are exactly the chunk ids j (ascending) with cluster_of_chunk[j]==c,
 * which is the reference's member order (build: invert_assignment ascending,
 * index.cpp:58-64; graft: push_back of increasing ids, streamer.cpp:130). */
typedef struct {
    uint32_t d;
    uint32_t n_tokens, cap_tokens, chunked_end;
    float* keys;   /* [cap_tokens*d] */
    float* values; /* [cap_tokens*d] */
    uint8_t* text_code; /* [cap_tokens] 0 "", 1 "\n", 2 "}" */
    uint32_t n_chunks, cap_chunks;
    uint32_t* chunk_start;      /* [cap_chunks] */
    uint32_t* chunk_end;        /* [cap_chunks] */
    uint32_t* chunk_kind;       /* [cap_chunks] BoundaryKind */
    uint32_t* chunk_level;      /* [cap_chunks] */
    float* chunk_rep;           /* [cap_chunks*d] */
    uint32_t* cluster_of_chunk; /* [cap_chunks] */
    uint32_t L;
    float* fine_centroid;        /* [L*d] */
    double* fine_radius;         /* [L] */
    uint64_t* fine_token_count;  /* [L] */
    uint32_t* fine_parent;       /* [L] */
    uint32_t* fine_member_count; /* [L] (chunks) */
    uint32_t P;
    float* coarse_centroid;      /* [P*d] */
    double* coarse_radius;       /* [P] */
    uint32_t* coarse_member_off; /* [P+1] */
    uint32_t* coarse_members;    /* fine ids, ascending within a unit */
    uint32_t structure_aware;    /* StreamerConfig::structure_aware */
    uint32_t graft_full;         /* GraftSearch::full */
} lco_index;

typedef struct { /* tierkv::Budgets (retriever.hpp:13-21) */
    uint32_t unit_topk;
    uint32_t mode; /* 0 fixed_cluster_count, 1 token_budget */
    uint32_t cluster_topk;
    uint64_t token_budget;
    uint32_t sink_size;
} lco_budgets;

typedef struct { /* tierkv::RetrievalResult (retriever.hpp:23-30) */
    uint32_t* units;    uint64_t n_units;    /* caller buffers, capacity >= P */
    uint32_t* clusters; uint64_t n_clusters; /* capacity >= L */
    uint32_t* active;   uint64_t n_active;   /* capacity >= n_tokens + n_buffer */
    float* output;                           /* [d] or NULL */
    uint64_t scanned;
    int degenerate;
} lco_result;

typedef struct { /* tierkv::GraftReport (streamer.hpp:27-35) */
    uint32_t chunk_id, cluster_id, unit_id;
    double centroid_delta, fine_radius, coarse_radius;
    uint64_t distance_comps;
} lco_graft_report;

/* status: 0 ok, 1 invalid_argument, 2 runtime_error */
/* FNV-1a-64 over raw bytes (the fixture fingerprint of SURVEY.md s8(d)) */
uint64_t lco_fnv1a64(const uint8_t* buf, size_t n);
double lco_dot(const float* a, const float* b, size_t d);     /* kernels.cpp:13-17 */
double lco_l2_norm(const float* a, size_t d);                 /* kernels.cpp:19-23 */
double lco_l2_dist(const float* a, const float* b, size_t d); /* kernels.cpp:25-32 */
void lco_upper_bounds(const float* q, const float* centroids, const double* radii, size_t n,
                      size_t d, double qnorm, double* scores); /* kernels.cpp:155-159 */
/* select_topk (retriever.cpp:27-39): ids sorted by (score desc, id asc), first k */
int lco_select_topk(const uint32_t* ids, const double* scores, size_t n, size_t k,
                    uint32_t* out, size_t* n_out);
int lco_attention(const float* q, const float* keys, const float* values, const uint32_t* ids,
                  size_t n_ids, size_t d, float* out); /* kernels.cpp:108-144 */
int lco_chunk_representative(const float* keys, size_t rows, size_t d, int max_pool,
                             float* out); /* index.cpp:20-41 */
int lco_retrieve(const lco_index* ix, const float* q, const lco_budgets* b,
                 const uint32_t* buffer, size_t n_buffer, int with_output,
                 lco_result* res); /* retriever.cpp:78-167 */
/* chunker segment() with ChunkPolicy::defaults() over text codes (chunker.cpp:103-149);
 * spans4 = (start, end, kind, level); returns span count */
size_t lco_segment_codes(const uint8_t* codes, size_t n, uint32_t* spans4);
/* push_token (streamer.cpp:56-66): returns 1 and fills span4 + rep when a chunk is emitted */
int lco_push_token(lco_index* ix, const float* key, const float* value, uint8_t code,
                   int* emitted, uint32_t* span4, float* rep);
int lco_graft_chunk(lco_index* ix, const uint32_t* span4, const float* rep,
                    lco_graft_report* rep_out); /* streamer.cpp:68-143 */
/* decode_step (streamer.cpp:145-165) minus the host stability metrics */
int lco_decode_step(lco_index* ix, const float* q, const float* key, const float* value,
                    uint8_t code, const lco_budgets* b, lco_result* res, int* grafted,
                    lco_graft_report* rep_out);

#ifdef __cplusplus
}
#endif
#endif
