/*
 * plaid_oracle.h — CPU restatement of the reference PLAID search path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker.  The product (paper_2205_09707_b200) never links it.
 *
 * Every function restates one reference function; the comment above each
 * definition in plaid_oracle.c cites /root/reference/proj/<file>:<line>.
 * Arithmetic follows the reference exactly (in-order fp32 sums, no FMA
 * contraction, fp64 norms), so on identical inputs the outputs are
 * bit-identical to the compiled reference (checked by tests/test_oracle.py
 * against oracle/_ref and the committed golden vectors in tests/golden/).
 *
 * Status codes: 0 = ok, otherwise lir::ErrorCode + 1 (error.hpp:8-26), the
 * same numbering as include/plaid.h.
 */
#ifndef PLAID_ORACLE_H
#define PLAID_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_index {
    uint32_t dim;
    uint32_t nbits;
    uint64_t num_centroids;   /* K */
    uint64_t num_passages;    /* N */
    uint64_t num_embeddings;  /* T */
    const float* centroids;   /* K x dim */
    const uint32_t* codes;    /* T */
    const uint8_t* residuals; /* T x nbits*dim/8 */
    const uint32_t* doclens;  /* N */
    const uint64_t* passage_offsets; /* N + 1 */
    const uint64_t* ivf_offsets;     /* K + 1 */
    const uint32_t* ivf_postings;
    const float* bucket_cutoffs;     /* 2^b - 1 */
    const float* bucket_weights;     /* 2^b */
} orc_index;

typedef struct orc_params {
    uint64_t k;
    uint64_t nprobe;
    float t_cs;
    uint64_t ndocs;
    int32_t disable_filter;
} orc_params;

/* Counter fields of lir::StageTrace (pipeline.hpp:23-43). */
typedef struct orc_trace {
    uint64_t stage1_candidates;
    uint64_t stage2_out;
    uint64_t stage3_out;
    uint64_t final_out;
    uint64_t centroid_matmul_count;
    uint64_t stage2_rows_gathered;
    uint64_t stage3_rows_gathered;
    uint64_t decompressed_passages;
} orc_trace;

const char* orc_last_error(void);

int orc_validate_query(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim);
int orc_validate_params(const orc_params* p, uint64_t num_centroids);
void orc_default_params_for_k(uint64_t k, orc_params* out);
uint64_t orc_stage3_width(const orc_params* p);

int orc_lut_build(uint32_t nbits, uint8_t* table /* 256 x 8/nbits */);
int orc_pack_residual(const uint8_t* idx, uint64_t n, uint32_t nbits, uint8_t* out);
int orc_unpack_via_lut(const uint8_t* packed, uint64_t n, uint32_t nbits, uint8_t* out);
int orc_reconstruct(const uint32_t* codes, uint64_t n, const uint8_t* residuals,
                    const float* centroids, uint32_t dim, uint32_t nbits,
                    const float* weights, float* out);

int orc_compute_centroid_scores(const float* q, uint64_t rows, uint64_t dim,
                                const float* centroids, uint64_t num_centroids,
                                float* scores, float* row_max);
int orc_generate_candidates(const float* scores, uint64_t num_centroids, uint64_t rows,
                            const uint64_t* ivf_offsets, const uint32_t* ivf_postings,
                            uint64_t nprobe, uint64_t num_passages,
                            uint32_t* out_ids, uint64_t* out_n);
void orc_prune_centroids(const float* row_max, uint64_t num_centroids, float t_cs, uint8_t* keep);
int orc_centroid_interaction(const orc_index* idx, const float* scores, uint64_t rows,
                             const uint32_t* cand, uint64_t n, const uint8_t* mask,
                             float* out_scores, uint64_t* rows_gathered);
int orc_select_top(const uint32_t* ids, const float* scores, uint64_t n, uint64_t keep,
                   uint32_t* out_ids, float* out_scores, uint64_t* out_n);
int orc_maxsim_packed(const float* scores, uint64_t nq, const uint64_t* offsets, uint64_t np,
                      float* out);
int orc_maxsim_embeddings(const float* q, uint64_t rows, uint64_t dim, const float* emb,
                          const uint64_t* offsets, uint64_t np, float* out);
int orc_rank_final(const orc_index* idx, const float* q, uint64_t rows,
                   const uint32_t* cand, uint64_t n, uint64_t k,
                   uint32_t* out_ids, float* out_scores, uint64_t* out_n);
int orc_search(const orc_index* idx, const float* q, uint64_t rows, uint64_t dim,
               const orc_params* p, uint32_t* out_ids, float* out_scores, uint64_t* out_n,
               orc_trace* trace);

#ifdef __cplusplus
}
#endif
#endif
