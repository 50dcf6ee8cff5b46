/*
 * plaid.h — C ABI of the B200-native PLAID searcher (libplaid.so).
 *
 * Drop-in boundary for the reference C++ searcher `lir` (/root/reference/proj).
 * Plain pointers and sizes only; no CUDA or torch types in any signature
 * (streams and device pointers travel as void* / uint64 where needed).
 *
 * Every entry point names the reference interface it replaces
 * (include/lir/<file>:<line>).  Status codes mirror lir::ErrorCode
 * (error.hpp:8-26) shifted by one, plus CUDA/NCCL/unsupported codes; a
 * thread-local message is available from plaid_last_error().
 *
 * Arithmetic contract: integer outputs (candidate sets, pruning masks, unpacked
 * residual indices, selections) are bit-exact with the reference on identical
 * inputs.  In PLAID_SCORES_EXACT mode every fp32 score is bit-exact too; in
 * PLAID_SCORES_TENSOR mode (tcgen05 S_cq) centroid scores are within ~1e-6
 * absolute and MaxSim scores within 1e-4 relative.
 */
#ifndef PLAID_H
#define PLAID_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLAID_ABI_VERSION 1

/* lir::ErrorCode (error.hpp:8-26) + 1. */
typedef enum plaid_status {
    PLAID_OK = 0,
    PLAID_DIMENSION_MISMATCH = 1,
    PLAID_NOT_NORMALIZED = 2,
    PLAID_TOO_FEW_POINTS = 3,
    PLAID_PACKING_UNSUPPORTED = 4,
    PLAID_EMPTY_CORPUS = 5,
    PLAID_INDEX_OUT_OF_RANGE = 6,
    PLAID_LENGTH_NOT_PACKABLE = 7,
    PLAID_EMPTY_PASSAGE_RANGE = 8,
    PLAID_INVALID_PARAMS = 9,
    PLAID_CHECKSUM_MISMATCH = 10,
    PLAID_UNSUPPORTED_VERSION = 11,
    PLAID_INVARIANT_VIOLATION = 12,
    PLAID_HEADER_MISMATCH = 13,
    PLAID_NORMALIZATION_ERROR = 14,
    PLAID_LENGTH_MISMATCH = 15,
    PLAID_UNKNOWN_QUERY_ID = 16,
    PLAID_IO_ERROR = 17,
    PLAID_CUDA_ERROR = 100,
    PLAID_NCCL_ERROR = 101,
    PLAID_UNSUPPORTED = 102,  /* outside the engine's envelope, e.g. |Q| > 32 */
    PLAID_OUT_OF_MEMORY = 103
} plaid_status;

typedef enum plaid_score_mode {
    PLAID_SCORES_TENSOR = 0, /* tcgen05 3xTF32 S_cq GEMM (production default) */
    PLAID_SCORES_EXACT = 1   /* in-order fp32 CUDA-core S_cq, bit-exact with lir */
} plaid_score_mode;

typedef struct plaid_index plaid_index;       /* device-resident CompressedIndex */
typedef struct plaid_searcher plaid_searcher; /* stream + scratch, one per host thread */

/* Mirrors lir::CompressedIndex's persisted fields (index.hpp:61-72). */
typedef struct plaid_index_desc {
    uint32_t dim;
    uint32_t nbits;
    uint64_t num_centroids;          /* K */
    uint64_t num_passages;           /* N */
    uint64_t num_embeddings;         /* T = sum(doclens) */
    const float* centroids;          /* K x dim, row-major, unit rows */
    const uint32_t* codes;           /* T */
    const uint8_t* residuals;        /* T x nbits*dim/8, LSB-first packing */
    const uint32_t* doclens;         /* N */
    const uint64_t* ivf_offsets;     /* K + 1 */
    const uint32_t* ivf_postings;    /* ivf_offsets[K], sorted unique per centroid */
    const float* bucket_cutoffs;     /* 2^nbits - 1 */
    const float* bucket_weights;     /* 2^nbits */
} plaid_index_desc;

/* lir::SearchParams (types.hpp:79-84) + SearchOptions.disable_filter (pipeline.hpp:45-48). */
typedef struct plaid_params {
    uint64_t k;
    uint64_t nprobe;
    float t_cs;
    uint64_t ndocs;
    int32_t disable_filter;
} plaid_params;

/* lir::StageTrace (pipeline.hpp:23-43): counters bit-exact, times from CUDA events. */
typedef struct plaid_trace {
    uint64_t stage1_candidates;
    uint64_t stage2_out;
    uint64_t stage3_out;
    uint64_t final_out;
    uint64_t centroid_matmul_count;
    uint64_t stage2_rows_gathered;
    uint64_t stage3_rows_gathered;
    uint64_t decompressed_passages;
    double candidate_generation_ms;
    double stage2_ms;
    double stage3_ms;
    double lookup_ms;
    double decompression_ms;
    double scoring_ms;
    double total_ms;
    uint64_t decompressed_tokens;  /* stage-4 tokens (sum of the finalists' doclens; not a lir counter) */
} plaid_trace;

typedef struct plaid_searcher_config {
    int32_t score_mode;     /* plaid_score_mode */
    int32_t record_times;   /* fill the *_ms fields of plaid_trace (adds events) */
    int32_t use_graphs;     /* plaid_search: capture H2D + launches + read-back as one CUDA graph per (rows, params), replay after */
    int32_t batch_engine;   /* plaid_batch_*: plaid_batch_engine */
} plaid_searcher_config;

/* Throughput-mode engine of plaid_batch_*: waves (one S_cq pass per wave of
 * queries + one CTA per query for stages 1b-4; used when the shape allows:
 * d = 128, |Q| <= 32, nprobe <= 8, filter on, stage3_width <= 2048) with the
 * lanes as fallback, or lanes only. */
typedef enum plaid_batch_engine { PLAID_BATCH_AUTO = 0, PLAID_BATCH_LANES = 1 } plaid_batch_engine;

/* ---- errors / host-side helpers ------------------------------------------------ */
const char* plaid_last_error(void);
const char* plaid_status_name(int status);              /* error.hpp:28-49 */
int plaid_abi_version(void);

/* types.cpp:61-72 validate_query; types.cpp:88-99 validate_params */
plaid_status plaid_validate_query(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim);
plaid_status plaid_validate_params(const plaid_params* p, uint64_t num_centroids);
/* types.cpp:74-86 */
void plaid_default_params_for_k(uint64_t k, plaid_params* out);
/* pipeline.cpp:227-230 */
uint64_t plaid_stage3_width(const plaid_params* p);

/* ---- index lifecycle ------------------------------------------------------------ */
/* Builds the device index from host arrays (index.hpp:60-85 + finalize_derived,
 * index.cpp:7-10).  validate != 0 runs validate_index's invariants (index.cpp:12-84). */
plaid_status plaid_index_from_host(const plaid_index_desc* desc, int device, int validate,
                                   plaid_index** out);
/* ---- on-disk index (SPEC.md storage module; layout in FORMAT.md) ----
 * plaid_index_save writes manifest.json + centroids.f32, codes.u32,
 * residuals.bin, doclens.u32, ivf_offsets.u64, ivf_postings.u32 (little
 * endian) with per-file checksums; on any write error the partial files are
 * removed (IoError).  Host-only: needs no GPU.
 * plaid_index_open maps the files, uploads them once to HBM and verifies every
 * checksum ON THE GPU over the uploaded arrays (ChecksumMismatch names the
 * file); UnsupportedVersion / HeaderMismatch / LengthMismatch for a bad
 * manifest; PLAID_OPEN_VALIDATE adds validate_index (index.cpp:12-84). */
enum { PLAID_OPEN_VALIDATE = 1, PLAID_OPEN_NO_CHECKSUMS = 2 };
plaid_status plaid_index_save(const plaid_index_desc* desc, const char* dir, uint64_t rng_seed);
plaid_status plaid_index_open(const char* dir, int device, uint32_t flags, plaid_index** out);
/* Best-of-iters GB/s of a plain coalesced HBM read of `bytes` (L2 flushed
 * before each pass): the achievable streaming rate for a one-pass kernel of
 * that size (bench.py reports the S_cq kernel against it and against the copy
 * peak).  Returns a cudaError_t value (0 = ok). */
int plaid_measure_read_gbs(int device, uint64_t bytes, int iters, double* out_gbs);
/* FORMAT.md digest of a host buffer (the manifest's per-file checksum). */
uint64_t plaid_checksum(const void* data, uint64_t bytes);

/* Same, for a desc that already is one passage-range shard of a larger index
 * (local ids, local IVF): results report local id + pid_base. */
plaid_status plaid_index_from_host_at(const plaid_index_desc* desc, uint64_t pid_base, int device,
                                      plaid_index** out);
/* Passage-range shard [pid_begin, pid_end) of a host index: local IVF with
 * local ids; search results report global ids (local + pid_begin). */
plaid_status plaid_index_from_host_shard(const plaid_index_desc* desc, uint64_t pid_begin,
                                         uint64_t pid_end, int device, plaid_index** out);
/* The synthetic benchmark corpus generated directly in HBM:
 * passages [pid_base, pid_base + num_passages) of the corpus the host
 * generator defines (same SplitMix64 streams: identical integer arrays),
 * local IVF built on the device, results report global ids.  For corpora
 * that do not fit host memory (BASELINE configs[4]: 140M passages, ~45 GB
 * per shard of 8).  Fixture infrastructure, not part of the lir API. */
typedef struct plaid_synth_desc {
    uint64_t num_passages, num_centroids, pid_base, seed;
    uint32_t dim, nbits, mean_len, spread;
    double repeat;  /* probability that a token repeats an earlier code of its passage */
} plaid_synth_desc;
plaid_status plaid_index_synth(const plaid_synth_desc* desc, int device, plaid_index** out);
/* nq x qlen x dim unit-norm queries near reconstructed tokens of the index
 * (the host generator's query recipe), into host memory. */
plaid_status plaid_index_synth_queries(plaid_index* index, uint64_t nq, uint32_t qlen, double noise, uint64_t seed,
                                       float* out);
/* Copies the device arrays back (any pointer may be NULL); sizes from plaid_index_info. */
plaid_status plaid_index_export(plaid_index* index, float* centroids, uint32_t* codes, uint8_t* residuals,
                                uint32_t* doclens, uint64_t* ivf_offsets, uint32_t* ivf_postings, float* cutoffs,
                                float* weights);
/* Re-checks validate_index's invariants on the device copy (index.cpp:12-84). */
plaid_status plaid_index_validate(plaid_index* index);
void plaid_index_close(plaid_index* index);
/* dim, nbits, K, N, T, P, pid_base, device bytes */
void plaid_index_info(const plaid_index* index, uint64_t out[8]);

/* ---- search ----------------------------------------------------------------------- */
/* index may be NULL for the index-free kernels (select/unpack/maxsim). */
plaid_status plaid_searcher_create(plaid_index* index, int device, const plaid_searcher_config* cfg,
                                   plaid_searcher** out);
void plaid_searcher_destroy(plaid_searcher* s);

/* lir::search (pipeline.hpp:86-87 / pipeline.cpp:232-283).  Q is host memory,
 * rows x dim fp32.  out_pids / out_scores hold >= params->k entries, sorted by
 * (score desc, pid asc).  trace may be NULL.  Synchronous. */
plaid_status plaid_search(plaid_searcher* s, const float* q, uint64_t rows, uint64_t dim,
                          const plaid_params* params, uint32_t* out_pids, float* out_scores,
                          uint64_t* out_n, plaid_trace* trace);
/* nq queries [nq][rows][dim]; outputs [nq][k] and out_n[nq]; traces[nq] or NULL. */
plaid_status plaid_search_batch(plaid_searcher* s, const float* q, uint64_t nq, uint64_t rows,
                                uint64_t dim, const plaid_params* params, uint32_t* out_pids,
                                float* out_scores, uint64_t* out_n, plaid_trace* traces);
/* Device-resident variant: d_q [nq][rows][dim] on the searcher's device,
 * outputs d_pids/d_scores [nq][k], d_n [nq] on device, enqueued on `stream`
 * (a cudaStream_t, 0 = the searcher's own stream) and NOT synchronised.
 * Query norms are checked on the device; a failure is reported by the next
 * plaid_searcher_sync().  Used by bench.py for the HBM-resident timing. */
plaid_status plaid_search_device(plaid_searcher* s, const float* d_q, uint64_t nq, uint64_t rows,
                                 uint64_t dim, const plaid_params* params, uint32_t* d_pids,
                                 float* d_scores, uint64_t* d_n, uint64_t stream);
plaid_status plaid_searcher_sync(plaid_searcher* s);
/* Number of kernels the last search enqueued (for the bench's gpu_launches). */
uint64_t plaid_searcher_last_launches(const plaid_searcher* s);
/* CUDA-event durations (ms) of the last enqueued query's phases, measured on
 * the launching stream (record_times must be set): [0] S_cq kernel,
 * [1] top-nprobe + candidate generation, [2] stage-2 interaction, [3] stage-2
 * select, [4] stage 3, [5] stage-4 decompress+MaxSim kernel, [6] final top-k. */
plaid_status plaid_searcher_phase_ms(plaid_searcher* s, double out[7]);

/* Merge G per-shard top-k lists (score desc, pid asc) into the global top-k —
 * the final select after the NCCL all-gather. Host arrays. */
plaid_status plaid_merge_topk(plaid_searcher* s, const uint32_t* pids, const float* scores,
                              const uint64_t* counts, uint64_t shards, uint64_t stride, uint64_t k,
                              uint32_t* out_pids, float* out_scores, uint64_t* out_n);
/* Same on device buffers, enqueued on stream (0 = searcher stream). */
plaid_status plaid_merge_topk_device(plaid_searcher* s, const uint32_t* d_pids,
                                     const float* d_scores, const uint64_t* d_counts,
                                     uint64_t shards, uint64_t stride, uint64_t k, uint32_t* d_out_pids,
                                     float* d_out_scores, uint64_t* d_out_n, uint64_t stream);

/* ---- encode on the GPU -----------------------------------------
 * Given trained centroids and quantizer, what lir::build_index derives from
 * them (indexer.cpp:197-282): codes = assign_codes (exact in-order fp32 dots,
 * first max wins), residuals = quantise + LSB-first pack, the IVF =
 * build_inverted_list.  Bit-identical to the reference.  Host buffers in and
 * out; the embeddings are T x dim unit rows (NotNormalized otherwise). */
typedef struct plaid_encode_desc {
    uint32_t dim;
    uint32_t nbits;
    uint64_t num_centroids;       /* K */
    uint64_t num_passages;        /* N */
    uint64_t num_embeddings;      /* T = sum(doclens) */
    const float* embeddings;      /* T x dim */
    const uint32_t* doclens;      /* N */
    const float* centroids;       /* K x dim */
    const float* bucket_cutoffs;  /* 2^nbits - 1 */
} plaid_encode_desc;
plaid_status plaid_encode(const plaid_encode_desc* in, int device, uint32_t* codes, uint8_t* residuals,
                          uint64_t* ivf_offsets, uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings);

/* ---- full index build on the GPU: lir::build_index (indexer.cpp:197-282) --------------
 * Training sample (uniform, <= 2^20 rows, seeded partial Fisher-Yates), k-means++
 * seeding and Lloyd iterations (kmeans.cpp:78-175), assign_codes, the quantizer
 * fit (indexer.cpp:74-147), residual packing and the IVF — bit-identical to
 * the reference's build for the same corpus, config and seed.  The heavy loops
 * (seeding dots, every T x K assignment, the mean sums) run on the GPU; the
 * seed-driven sequential choices (k-means++ picks, empty-cluster repair, the
 * quantizer's pool statistics) stay on the host in the reference's order.
 * num_centroids 0 = auto_num_centroids (2^ceil(log2(T)/2)); centroids_cap
 * rows must hold the resulting K (checked); ivf_offsets has K + 1 entries. */
typedef struct plaid_build_desc {
    uint32_t dim;
    uint32_t nbits;
    uint64_t num_passages;     /* N */
    uint64_t num_embeddings;   /* T = sum(doclens) */
    const float* embeddings;   /* T x dim, unit rows */
    const uint32_t* doclens;   /* N */
    uint64_t num_centroids;    /* 0 = auto */
    uint64_t kmeans_iters;     /* IndexConfig::kmeans_iters (reference default 20) */
    uint64_t rng_seed;         /* IndexConfig::rng_seed (reference default 42) */
} plaid_build_desc;
plaid_status plaid_build_index(const plaid_build_desc* in, int device, float* centroids, uint64_t centroids_cap,
                               uint64_t* num_centroids, float* bucket_cutoffs, float* bucket_weights, uint32_t* codes,
                               uint8_t* residuals, uint64_t* ivf_offsets, uint32_t* ivf_postings, uint64_t postings_cap,
                               uint64_t* num_postings);

/* ---- throughput mode (BASELINE configs[2]: batched queries) ---------------------------
 * `lanes` searchers (own CUDA stream + scratch each) over one index; query j of
 * a batch runs on lane j mod lanes, so the stages of different queries overlap
 * on the GPU.  Results are identical to plaid_search per query. */
typedef struct plaid_batch plaid_batch;
plaid_status plaid_batch_create(plaid_index* index, int device, const plaid_searcher_config* cfg, uint32_t lanes,
                                plaid_batch** out);
void plaid_batch_destroy(plaid_batch* b);
/* Host buffers: q [nq][rows][dim]; out_pids / out_scores [nq][k]; out_n [nq].
 * Every query is validated before any work (types.cpp:61-99).  Synchronous. */
plaid_status plaid_batch_search(plaid_batch* b, const float* q, uint64_t nq, uint64_t rows, uint64_t dim,
                                const plaid_params* params, uint32_t* out_pids, float* out_scores, uint64_t* out_n);
/* Device buffers, forked from and joined back to `stream` (0 = lane 0's);
 * not synchronised (query norms are checked on the device, reported by
 * plaid_batch_sync). */
plaid_status plaid_batch_search_device(plaid_batch* b, const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim,
                                       const plaid_params* params, uint32_t* d_pids, float* d_scores, uint64_t* d_n,
                                       uint64_t stream);
plaid_status plaid_batch_sync(plaid_batch* b);
uint64_t plaid_batch_last_launches(const plaid_batch* b);
/* After a batch that ran on the wave engine: per query [stage1_candidates,
 * stage2_out, stage3_out, final_out] (lir::StageTrace counters), out[nq][4].
 * Synchronises.  PLAID_INVALID_PARAMS when the last batch ran on lanes. */
plaid_status plaid_batch_counters(plaid_batch* b, uint64_t* out, uint64_t nq);
/* Test hook: the S_cq table (num_centroids x 32 floats, one row per
 * centroid) the last wave computed for its j-th query (j < wave size). */
plaid_status plaid_batch_wave_scores(plaid_batch* b, uint64_t j, float* out);
/* Queries per wave of the wave engine (0 before its first batch). */
uint32_t plaid_batch_wave_slots(const plaid_batch* b);
/* 1 when the last batch ran on the wave engine, else 0. */
int plaid_batch_last_was_wave(const plaid_batch* b);

/* ---- global-exact passage-sharded search ----------------------------
 * The reference searches one index (pipeline.cpp:232-283); a passage-range
 * shard alone cannot know the global stage-2 (top-ndocs) and stage-3
 * (top-stage3_width) cuts.  Each shard runs three enqueue-only phases on its
 * searcher; between them the caller all-gathers every shard's exported key row
 * (u64, zero-padded to a stride common to all shards, e.g. NCCL all-gather):
 *   phase1: stages 1-2 -> d_x2[stride2] = this shard's top-ndocs keys
 *           (stride2 >= min(ndocs, shard N); the global min(ndocs, N) works)
 *   phase2: d_g2[shards * stride2] -> keep only the global top-ndocs members,
 *           stage 3 -> d_x3[stride3] (stride3 >= min(stage3_width, shard N))
 *   phase3: d_g3[shards * stride3] -> keep the global stage-3 members, stage 4,
 *           this shard's top-k (global pids) into d_pids/d_scores/d_n.
 * Merging the shards' top-k (plaid_merge_topk_device) then equals lir::search
 * over the unsharded index, and the per-shard trace counters
 * (plaid_searcher_trace_counters_device) sum to its StageTrace counters.
 * With disable_filter the exports are skipped (nothing is cut before stage 4). */
plaid_status plaid_shard_phase1_device(plaid_searcher* s, const float* d_q, uint64_t rows, uint64_t dim,
                                       const plaid_params* params, uint64_t* d_x2, uint64_t stride2,
                                       uint64_t stream);
plaid_status plaid_shard_phase2_device(plaid_searcher* s, const uint64_t* d_g2, uint64_t shards,
                                       uint64_t* d_x3, uint64_t stride3, uint64_t stream);
plaid_status plaid_shard_phase3_device(plaid_searcher* s, const uint64_t* d_g3, uint64_t shards,
                                       uint32_t* d_pids, float* d_scores, uint64_t* d_n, uint64_t stream);
/* d_out[6] <- [stage1_candidates, stage2_out, stage3_out, final_out (host path
 * only), stage2_rows_gathered, stage3_rows_gathered] of the last query. */
plaid_status plaid_searcher_trace_counters_device(plaid_searcher* s, uint64_t* d_out, uint64_t stream);

/* Same from packed rows, one all-gather per query: row g (of `shards`) at
 * d_rows + g * (2k + 2) u32 words = [k u32 pids | k f32 scores | u64 count]
 * (what plaid_shard_phase3_device / plaid_search_device write when given
 * pids = row, scores = row + k, n = (uint64_t*)(row + 2k)). */
plaid_status plaid_merge_topk_rows_device(plaid_searcher* s, const uint32_t* d_rows, uint64_t shards, uint64_t k,
                                          uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n,
                                          uint64_t stream);

/* Batched form for throughput mode over passage shards: pids/scores
 * [shards][B][k] and counts [shards][B] (e.g. one NCCL all-gather of every
 * shard's [B][k] results) -> out [B][k] + out_n[B], one kernel for the whole
 * batch.  shards * k <= 25600. */
plaid_status plaid_merge_topk_batch_device(plaid_searcher* s, const uint32_t* d_pids, const float* d_scores,
                                           const uint64_t* d_counts, uint64_t shards, uint64_t batch, uint64_t k,
                                           uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n,
                                           uint64_t stream);

/* ---- single-process sharded search over several GPUs -------------
 * The drop-in for lir::search (pipeline.hpp:86-87) over a passage-sharded
 * index: `shards` are disjoint passage ranges (plaid_index_from_host_shard /
 * _at, each on its own GPU or sharing one), searched by one searcher per
 * shard on its device; the exchanges are on-device all-gathers that read the
 * other shards' rows through NVLink peer access (no host round trip), and the
 * final select runs on shards[0]'s device.  mode GLOBAL_EXACT reproduces
 * lir::search over the unsharded index (ids, scores, trace counters summed);
 * SHARD_LOCAL is the reference run per shard followed by the top-k merge.
 * Synchronous, host buffers like plaid_search. */
typedef struct plaid_sharded plaid_sharded;
enum { PLAID_SHARD_GLOBAL_EXACT = 0, PLAID_SHARD_LOCAL = 1 };
plaid_status plaid_sharded_create(plaid_index* const* shards, uint32_t num_shards, const plaid_searcher_config* cfg,
                                  int32_t mode, plaid_sharded** out);
void plaid_sharded_destroy(plaid_sharded* s);
plaid_status plaid_sharded_search(plaid_sharded* s, const float* q, uint64_t rows, uint64_t dim,
                                  const plaid_params* params, uint32_t* out_pids, float* out_scores, uint64_t* out_n,
                                  plaid_trace* trace);
uint64_t plaid_sharded_last_launches(const plaid_sharded* s);

/* ---- per-stage entry points (host buffers in/out, computed on the GPU) ------------ */
/* pipeline.cpp:26-50: scores K x rows (centroid-major), row_max K */
plaid_status plaid_compute_centroid_scores(plaid_searcher* s, const float* q, uint64_t rows,
                                           uint64_t dim, float* scores, float* row_max);
/* pipeline.cpp:52-87: scores K x rows from the host; out_ids sorted ascending (capacity N) */
plaid_status plaid_generate_candidates(plaid_searcher* s, const float* scores, uint64_t rows,
                                       uint64_t nprobe, uint32_t* out_ids, uint64_t* out_n);
/* pipeline.cpp:89-95 */
plaid_status plaid_prune_centroids(plaid_searcher* s, const float* row_max, uint64_t num_centroids,
                                   float t_cs, uint8_t* keep);
/* pipeline.cpp:97-137: mask may be NULL */
plaid_status plaid_centroid_interaction(plaid_searcher* s, const float* scores, uint64_t rows,
                                        const uint32_t* cand, uint64_t n, const uint8_t* mask,
                                        float* out_scores, uint64_t* rows_gathered);
/* pipeline.cpp:139-163 */
plaid_status plaid_select_top(plaid_searcher* s, const uint32_t* ids, const float* scores,
                              uint64_t n, uint64_t keep, uint32_t* out_ids, float* out_scores,
                              uint64_t* out_n);
/* pipeline.cpp:165-225 */
plaid_status plaid_rank_final(plaid_searcher* s, const float* q, uint64_t rows,
                              const uint32_t* cand, uint64_t n, uint64_t k, uint32_t* out_ids,
                              float* out_scores, uint64_t* out_n);
/* residual_codec.cpp:97-132 (uses the index's centroids and quantizer) */
plaid_status plaid_reconstruct(plaid_searcher* s, const uint32_t* codes, uint64_t n,
                               const uint8_t* residuals, float* out);
/* residual_codec.cpp:42-59 / :86-95 */
plaid_status plaid_lut_build(uint32_t nbits, uint8_t* table);
plaid_status plaid_unpack_via_lut(plaid_searcher* s, const uint8_t* packed, uint64_t n,
                                  uint32_t nbits, uint8_t* out);
/* residual_codec.cpp:61-84 (host; index-build side, kept for round trips) */
plaid_status plaid_pack_residual(const uint8_t* idx, uint64_t n, uint32_t nbits, uint8_t* out);
/* maxsim.cpp:31-64 */
plaid_status plaid_maxsim_packed(plaid_searcher* s, const float* scores, uint64_t nq,
                                 const uint64_t* offsets, uint64_t np, float* out);
/* maxsim.cpp:66-104 */
plaid_status plaid_maxsim_embeddings(plaid_searcher* s, const float* q, uint64_t rows, uint64_t dim,
                                     const float* emb, const uint64_t* offsets, uint64_t np,
                                     float* out);

#ifdef __cplusplus
}
#endif
#endif /* PLAID_H */
