/*
 * plaid_oracle.c — CPU restatement of the reference PLAID four-stage search.
 *
 * TEST INFRASTRUCTURE ONLY (see plaid_oracle.h).  Not linked by the product.
 * Compiled with -O2 -ffp-contract=off so every fp32 expression rounds exactly
 * like the reference's in-order loops (types.hpp:18-22 `dot`).
 *
 * Citations are /root/reference/proj/<file>:<line>.
 */
#include "plaid_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* lir::ErrorCode (error.hpp:8-26) + 1; 0 = ok. */
enum {
    ORC_OK = 0,
    ORC_DimensionMismatch = 1,
    ORC_NotNormalized = 2,
    ORC_TooFewPoints = 3,
    ORC_PackingUnsupported = 4,
    ORC_EmptyCorpus = 5,
    ORC_IndexOutOfRange = 6,
    ORC_LengthNotPackable = 7,
    ORC_EmptyPassageRange = 8,
    ORC_InvalidParams = 9,
    ORC_ChecksumMismatch = 10,
    ORC_UnsupportedVersion = 11,
    ORC_InvariantViolation = 12,
    ORC_HeaderMismatch = 13,
    ORC_NormalizationError = 14,
    ORC_LengthMismatch = 15,
    ORC_UnknownQueryId = 16,
    ORC_IoError = 17,
    ORC_OutOfMemory = 102,
};

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* types.hpp:18-22 — in-order fp32 dot, no contraction. */
static float dot_f(const float* a, const float* b, uint64_t dim) {
    float acc = 0.0f;
    for (uint64_t i = 0; i < dim; ++i) acc += a[i] * b[i];
    return acc;
}

/* types.hpp:24-28 */
static double l2_norm(const float* v, uint64_t dim) {
    double acc = 0.0;
    for (uint64_t i = 0; i < dim; ++i) acc += (double)v[i] * (double)v[i];
    return sqrt(acc);
}

/* types.cpp:61-72 with check_unit_rows types.cpp:10-19, tolerance types.hpp:16 */
int orc_validate_query(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim) {
    if (rows == 0) return fail(ORC_InvalidParams, "query must contain at least one token");
    if (dim != index_dim) return fail(ORC_DimensionMismatch, "query dim does not match index dim");
    const double tol = (double)1e-3f;
    for (uint64_t r = 0; r < rows; ++r) {
        double norm = l2_norm(q + r * dim, dim);
        if (fabs(norm - 1.0) > tol) return fail(ORC_NotNormalized, "query row not unit norm");
    }
    return ORC_OK;
}

/* types.cpp:88-99 */
int orc_validate_params(const orc_params* p, uint64_t num_centroids) {
    if (p->k < 1) return fail(ORC_InvalidParams, "k must be >= 1");
    if (p->nprobe < 1 || p->nprobe > num_centroids) return fail(ORC_InvalidParams, "nprobe outside [1, K]");
    if (p->ndocs < p->k) return fail(ORC_InvalidParams, "ndocs must be >= k");
    if (!(p->t_cs >= -1.0f && p->t_cs <= 1.0f)) return fail(ORC_InvalidParams, "t_cs must lie in [-1, 1]");
    return ORC_OK;
}

/* types.cpp:74-86 */
void orc_default_params_for_k(uint64_t k, orc_params* out) {
    out->k = k;
    out->disable_filter = 0;
    if (k <= 10) {
        out->nprobe = 1; out->t_cs = 0.5f; out->ndocs = 256;
    } else if (k <= 100) {
        out->nprobe = 2; out->t_cs = 0.45f; out->ndocs = 1024;
    } else {
        out->nprobe = 4; out->t_cs = 0.4f; out->ndocs = 4096;
    }
    if (out->ndocs < k) out->ndocs = k;
}

/* pipeline.cpp:227-230 */
uint64_t orc_stage3_width(const orc_params* p) {
    uint64_t quarter = (p->ndocs + 3) / 4;
    return quarter > p->k ? quarter : p->k;
}

static int nbits_supported(uint32_t nbits) { return nbits == 1 || nbits == 2 || nbits == 4; }

/* residual_codec.cpp:42-59 — LSB-first table[v][j] = (v >> (b*j)) & (2^b-1). */
int orc_lut_build(uint32_t nbits, uint8_t* table) {
    if (!nbits_supported(nbits)) return fail(ORC_PackingUnsupported, "nbits not in {1,2,4}");
    uint32_t per = 8 / nbits;
    uint8_t mask = (uint8_t)((1u << nbits) - 1);
    for (unsigned v = 0; v < 256; ++v)
        for (uint32_t j = 0; j < per; ++j) table[v * per + j] = (uint8_t)((v >> (nbits * j)) & mask);
    return ORC_OK;
}

/* residual_codec.cpp:61-84 */
int orc_pack_residual(const uint8_t* idx, uint64_t n, uint32_t nbits, uint8_t* out) {
    if (!nbits_supported(nbits)) return fail(ORC_PackingUnsupported, "nbits not in {1,2,4}");
    uint32_t per = 8 / nbits;
    if (n % per != 0) return fail(ORC_LengthNotPackable, "indices not divisible by 8/nbits");
    memset(out, 0, n / per);
    for (uint64_t i = 0; i < n; ++i) {
        if (idx[i] >= (1u << nbits)) return fail(ORC_IndexOutOfRange, "bucket index out of range");
        out[i / per] |= (uint8_t)(idx[i] << (nbits * (i % per)));
    }
    return ORC_OK;
}

/* residual_codec.cpp:86-95 */
int orc_unpack_via_lut(const uint8_t* packed, uint64_t n, uint32_t nbits, uint8_t* out) {
    uint8_t table[256 * 8];
    int rc = orc_lut_build(nbits, table);
    if (rc) return rc;
    uint32_t per = 8 / nbits;
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < per; ++j) out[i * per + j] = table[packed[i] * per + j];
    return ORC_OK;
}

/* residual_codec.cpp:97-132 — v = C[code] + w[idx] (fp32), fp64 in-order norm,
 * inv = float(1/sqrt(norm^2)), v *= inv when norm^2 > 0. */
int orc_reconstruct(const uint32_t* codes, uint64_t n, const uint8_t* residuals,
                    const float* centroids, uint32_t dim, uint32_t nbits,
                    const float* weights, float* out) {
    uint8_t table[256 * 8];
    int rc = orc_lut_build(nbits, table);
    if (rc) return rc;
    const uint32_t per = 8 / nbits;
    const uint64_t bpt = (uint64_t)nbits * dim / 8;
    for (uint64_t t = 0; t < n; ++t) {
        const float* cent = centroids + (uint64_t)codes[t] * dim;
        const uint8_t* bytes = residuals + t * bpt;
        float* v = out + t * dim;
        uint64_t d = 0;
        for (uint64_t b = 0; b < bpt; ++b) {
            const uint8_t* row = table + bytes[b] * per;
            for (uint32_t j = 0; j < per; ++j, ++d) v[d] = cent[d] + weights[row[j]];
        }
        double norm_sq = 0.0;
        for (uint64_t i = 0; i < dim; ++i) norm_sq += (double)v[i] * (double)v[i];
        if (norm_sq > 0.0) {
            float inv = (float)(1.0 / sqrt(norm_sq));
            for (uint64_t i = 0; i < dim; ++i) v[i] *= inv;
        }
    }
    return ORC_OK;
}

/* pipeline.cpp:26-50 — S[c][i] = dot(C[c], Q[i]); row max initialised to -inf. */
int orc_compute_centroid_scores(const float* q, uint64_t rows, uint64_t dim,
                                const float* centroids, uint64_t num_centroids,
                                float* scores, float* row_max) {
    for (uint64_t c = 0; c < num_centroids; ++c) {
        const float* cent = centroids + c * dim;
        float* out = scores + c * rows;
        float mx = -INFINITY;
        for (uint64_t i = 0; i < rows; ++i) {
            float s = dot_f(cent, q + i * dim, dim);
            out[i] = s;
            if (s > mx) mx = s;
        }
        row_max[c] = mx;
    }
    return ORC_OK;
}

typedef struct { float s; uint32_t id; } scored_id;

/* (score desc, id asc) — pipeline.cpp:67-72 and :147-150.  Scores compare with
 * `!=`, so -0.0 and +0.0 are equal and fall through to the id. */
static int better(const scored_id* a, const scored_id* b) {
    if (a->s != b->s) return a->s > b->s;
    return a->id < b->id;
}

static int cmp_scored(const void* pa, const void* pb) {
    const scored_id* a = (const scored_id*)pa;
    const scored_id* b = (const scored_id*)pb;
    if (better(a, b)) return -1;
    if (better(b, a)) return 1;
    return 0;
}

/* pipeline.cpp:52-87 — per query token the nprobe best centroids by
 * (S desc, c asc); union of their postings; output sorted ascending. */
int orc_generate_candidates(const float* scores, uint64_t num_centroids, uint64_t rows,
                            const uint64_t* ivf_offsets, const uint32_t* ivf_postings,
                            uint64_t nprobe, uint64_t num_passages,
                            uint32_t* out_ids, uint64_t* out_n) {
    if (nprobe < 1 || nprobe > num_centroids) return fail(ORC_InvalidParams, "nprobe outside [1, K]");
    uint8_t* seen = (uint8_t*)calloc(num_passages ? num_passages : 1, 1);
    scored_id* best = (scored_id*)malloc(sizeof(scored_id) * (nprobe < num_centroids ? num_centroids : nprobe));
    if (!seen || !best) { free(seen); free(best); return fail(ORC_OutOfMemory, "oom"); }
    for (uint64_t i = 0; i < rows; ++i) {
        uint64_t nb = 0;
        if (nprobe <= 64) {
            /* bounded insertion keeps the nprobe best in order */
            for (uint64_t c = 0; c < num_centroids; ++c) {
                scored_id x = {scores[c * rows + i], (uint32_t)c};
                if (nb == nprobe && !better(&x, &best[nb - 1])) continue;
                uint64_t pos = nb < nprobe ? nb++ : nb - 1;
                while (pos > 0 && better(&x, &best[pos - 1])) { best[pos] = best[pos - 1]; --pos; }
                best[pos] = x;
            }
        } else {
            for (uint64_t c = 0; c < num_centroids; ++c) {
                best[c].s = scores[c * rows + i];
                best[c].id = (uint32_t)c;
            }
            qsort(best, num_centroids, sizeof(scored_id), cmp_scored);
            nb = nprobe;
        }
        for (uint64_t t = 0; t < nb; ++t) {
            uint32_t c = best[t].id;
            for (uint64_t j = ivf_offsets[c]; j < ivf_offsets[c + 1]; ++j) seen[ivf_postings[j]] = 1;
        }
    }
    /* std::sort of the unique ids (pipeline.cpp:83) == ascending scan of seen */
    uint64_t n = 0;
    for (uint64_t p = 0; p < num_passages; ++p)
        if (seen[p]) out_ids[n++] = (uint32_t)p;
    *out_n = n;
    free(seen);
    free(best);
    return ORC_OK;
}

/* pipeline.cpp:89-95 — keep[c] = row_max[c] >= t_cs (non-strict). */
void orc_prune_centroids(const float* row_max, uint64_t num_centroids, float t_cs, uint8_t* keep) {
    for (uint64_t c = 0; c < num_centroids; ++c) keep[c] = row_max[c] >= t_cs ? 1 : 0;
}

/* pipeline.cpp:97-137 — acc = -inf; fold S rows of (unmasked) codes with `>`;
 * total = in-order fp32 sum if any row was used, else 0. */
int orc_centroid_interaction(const orc_index* idx, const float* scores, uint64_t rows,
                             const uint32_t* cand, uint64_t n, const uint8_t* mask,
                             float* out_scores, uint64_t* rows_gathered) {
    if (n == 0) return fail(ORC_InvalidParams, "centroid interaction requires candidates");
    float acc[1024];
    if (rows > 1024) return fail(ORC_InvalidParams, "oracle supports |Q| <= 1024");
    uint64_t gathered = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t pid = cand[i];
        const uint32_t* codes = idx->codes + idx->passage_offsets[pid];
        uint32_t len = idx->doclens[pid];
        for (uint64_t j = 0; j < rows; ++j) acc[j] = -INFINITY;
        uint64_t used = 0;
        for (uint32_t t = 0; t < len; ++t) {
            uint32_t code = codes[t];
            if (mask && !mask[code]) continue;
            const float* row = scores + (uint64_t)code * rows;
            for (uint64_t j = 0; j < rows; ++j)
                if (row[j] > acc[j]) acc[j] = row[j];
            ++used;
        }
        gathered += used;
        float total = 0.0f;
        if (used > 0)
            for (uint64_t j = 0; j < rows; ++j) total += acc[j];
        out_scores[i] = total;
    }
    if (rows_gathered) *rows_gathered = gathered;
    return ORC_OK;
}

/* pipeline.cpp:139-163 */
int orc_select_top(const uint32_t* ids, const float* scores, uint64_t n, uint64_t keep,
                   uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    if (keep < 1) return fail(ORC_InvalidParams, "selection width must be >= 1");
    scored_id* a = (scored_id*)malloc(sizeof(scored_id) * (n ? n : 1));
    if (!a) return fail(ORC_OutOfMemory, "oom");
    for (uint64_t i = 0; i < n; ++i) { a[i].s = scores[i]; a[i].id = ids[i]; }
    qsort(a, n, sizeof(scored_id), cmp_scored);
    uint64_t m = keep < n ? keep : n;
    for (uint64_t i = 0; i < m; ++i) { out_ids[i] = a[i].id; out_scores[i] = a[i].s; }
    *out_n = m;
    free(a);
    return ORC_OK;
}

/* maxsim.cpp:11-27 */
static int check_offsets(const uint64_t* offsets, uint64_t np, uint64_t total_rows) {
    if (offsets[0] != 0) return fail(ORC_InvalidParams, "offsets must start at 0");
    for (uint64_t p = 0; p < np; ++p) {
        if (offsets[p + 1] < offsets[p]) return fail(ORC_InvalidParams, "offsets must be monotone");
        if (offsets[p + 1] == offsets[p]) return fail(ORC_EmptyPassageRange, "passage has no token rows");
    }
    if (offsets[np] != total_rows) return fail(ORC_LengthMismatch, "last offset does not match row count");
    return ORC_OK;
}

/* maxsim.cpp:31-64 */
int orc_maxsim_packed(const float* scores, uint64_t nq, const uint64_t* offsets, uint64_t np,
                      float* out) {
    if (nq == 0) return fail(ORC_InvalidParams, "need at least one query token");
    int rc = check_offsets(offsets, np, offsets[np]);
    if (rc) return rc;
    float acc[1024];
    if (nq > 1024) return fail(ORC_InvalidParams, "oracle supports |Q| <= 1024");
    for (uint64_t p = 0; p < np; ++p) {
        const float* row = scores + offsets[p] * nq;
        for (uint64_t i = 0; i < nq; ++i) acc[i] = row[i];
        uint64_t len = offsets[p + 1] - offsets[p];
        for (uint64_t t = 1; t < len; ++t) {
            row += nq;
            for (uint64_t i = 0; i < nq; ++i)
                if (row[i] > acc[i]) acc[i] = row[i];
        }
        float total = 0.0f;
        for (uint64_t i = 0; i < nq; ++i) total += acc[i];
        out[p] = total;
    }
    return ORC_OK;
}

/* maxsim.cpp:66-104 — acc initialised from the first token (:89). */
int orc_maxsim_embeddings(const float* q, uint64_t rows, uint64_t dim, const float* emb,
                          const uint64_t* offsets, uint64_t np, float* out) {
    if (rows == 0 || dim == 0) return fail(ORC_InvalidParams, "empty query matrix");
    int rc = check_offsets(offsets, np, offsets[np]);
    if (rc) return rc;
    float acc[1024];
    if (rows > 1024) return fail(ORC_InvalidParams, "oracle supports |Q| <= 1024");
    for (uint64_t p = 0; p < np; ++p) {
        const float* tok = emb + offsets[p] * dim;
        for (uint64_t i = 0; i < rows; ++i) acc[i] = dot_f(q + i * dim, tok, dim);
        uint64_t len = offsets[p + 1] - offsets[p];
        for (uint64_t t = 1; t < len; ++t) {
            tok += dim;
            for (uint64_t i = 0; i < rows; ++i) {
                float s = dot_f(q + i * dim, tok, dim);
                if (s > acc[i]) acc[i] = s;
            }
        }
        float total = 0.0f;
        for (uint64_t i = 0; i < rows; ++i) total += acc[i];
        out[p] = total;
    }
    return ORC_OK;
}

/* pipeline.cpp:165-225 — gather, reconstruct, maxsim_embeddings, select_top(k). */
int orc_rank_final(const orc_index* idx, const float* q, uint64_t rows,
                   const uint32_t* cand, uint64_t n, uint64_t k,
                   uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    if (n == 0) return fail(ORC_InvalidParams, "final ranking requires candidates");
    const uint64_t dim = idx->dim;
    const uint64_t bpt = (uint64_t)idx->nbits * dim / 8;
    uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
    if (!offsets) return fail(ORC_OutOfMemory, "oom");
    offsets[0] = 0;
    for (uint64_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + idx->doclens[cand[i]];
    uint64_t total = offsets[n];
    float* emb = (float*)malloc(sizeof(float) * (total ? total : 1) * dim);
    float* sc = (float*)malloc(sizeof(float) * n);
    if (!emb || !sc) { free(offsets); free(emb); free(sc); return fail(ORC_OutOfMemory, "oom"); }
    int rc = ORC_OK;
    for (uint64_t i = 0; i < n && !rc; ++i) {
        uint64_t src = idx->passage_offsets[cand[i]];
        rc = orc_reconstruct(idx->codes + src, idx->doclens[cand[i]], idx->residuals + src * bpt,
                             idx->centroids, idx->dim, idx->nbits, idx->bucket_weights,
                             emb + offsets[i] * dim);
    }
    if (!rc) rc = orc_maxsim_embeddings(q, rows, dim, emb, offsets, n, sc);
    if (!rc) rc = orc_select_top(cand, sc, n, k, out_ids, out_scores, out_n);
    free(offsets);
    free(emb);
    free(sc);
    return rc;
}

/* pipeline.cpp:232-283 */
int orc_search(const orc_index* idx, const float* q, uint64_t rows, uint64_t dim,
               const orc_params* p, uint32_t* out_ids, float* out_scores, uint64_t* out_n,
               orc_trace* trace) {
    orc_trace tr;
    memset(&tr, 0, sizeof tr);
    *out_n = 0;
    int rc = orc_validate_query(q, rows, dim, idx->dim);
    if (!rc) rc = orc_validate_params(p, idx->num_centroids);
    if (rc) { if (trace) *trace = tr; return rc; }

    const uint64_t K = idx->num_centroids, N = idx->num_passages;
    float* S = (float*)malloc(sizeof(float) * K * rows);
    float* rmax = (float*)malloc(sizeof(float) * K);
    uint32_t* c1 = (uint32_t*)malloc(sizeof(uint32_t) * (N ? N : 1));
    uint8_t* keep = (uint8_t*)malloc(K);
    float* sc = (float*)malloc(sizeof(float) * (N ? N : 1));
    uint32_t* k2 = (uint32_t*)malloc(sizeof(uint32_t) * (N ? N : 1));
    float* k2s = (float*)malloc(sizeof(float) * (N ? N : 1));
    uint32_t* k3 = (uint32_t*)malloc(sizeof(uint32_t) * (N ? N : 1));
    float* k3s = (float*)malloc(sizeof(float) * (N ? N : 1));
    if (!S || !rmax || !c1 || !keep || !sc || !k2 || !k2s || !k3 || !k3s) {
        rc = fail(ORC_OutOfMemory, "oom");
        goto done;
    }
    orc_compute_centroid_scores(q, rows, dim, idx->centroids, K, S, rmax);
    tr.centroid_matmul_count = 1;
    uint64_t n1 = 0;
    rc = orc_generate_candidates(S, K, rows, idx->ivf_offsets, idx->ivf_postings, p->nprobe, N, c1, &n1);
    if (rc) goto done;
    tr.stage1_candidates = n1;
    if (n1 == 0) goto done;

    const uint32_t* fin = c1;
    uint64_t nfin = n1;
    if (p->disable_filter) {
        tr.stage2_out = n1;
        tr.stage3_out = n1;
    } else {
        orc_prune_centroids(rmax, K, p->t_cs, keep);
        rc = orc_centroid_interaction(idx, S, rows, c1, n1, keep, sc, &tr.stage2_rows_gathered);
        if (rc) goto done;
        uint64_t n2 = 0;
        rc = orc_select_top(c1, sc, n1, p->ndocs, k2, k2s, &n2);
        if (rc) goto done;
        tr.stage2_out = n2;
        rc = orc_centroid_interaction(idx, S, rows, k2, n2, NULL, sc, &tr.stage3_rows_gathered);
        if (rc) goto done;
        uint64_t n3 = 0;
        rc = orc_select_top(k2, sc, n2, orc_stage3_width(p), k3, k3s, &n3);
        if (rc) goto done;
        tr.stage3_out = n3;
        fin = k3;
        nfin = n3;
    }
    rc = orc_rank_final(idx, q, rows, fin, nfin, p->k, out_ids, out_scores, out_n);
    if (rc) goto done;
    tr.decompressed_passages = nfin;
    tr.final_out = *out_n;
done:
    if (trace) *trace = tr;
    free(S); free(rmax); free(c1); free(keep); free(sc); free(k2); free(k2s); free(k3); free(k3s);
    return rc;
}
