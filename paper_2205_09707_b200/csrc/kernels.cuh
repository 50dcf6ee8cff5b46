// kernels.cuh — launchers for the PLAID search kernels (sm_100a).
//
// All kernels are enqueued on an explicit stream and read data-dependent
// sizes (candidate counts) from device memory, so a whole search is a fixed
// launch sequence that can be captured in a CUDA graph with no host sync.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace plaid {

// Device view of a CompressedIndex (index.hpp:60-85) + derived arrays.
struct IndexView {
    uint32_t dim = 0;
    uint32_t nbits = 0;
    uint64_t K = 0, N = 0, T = 0, P = 0;
    uint32_t max_doclen = 0;
    const float* centroids = nullptr;   // K x dim
    const uint32_t* codes = nullptr;    // T
    const uint8_t* residuals = nullptr; // T x nbits*dim/8
    const uint32_t* doclens = nullptr;  // N
    const uint64_t* offsets = nullptr;  // N + 1
    const uint64_t* ivf_offsets = nullptr;
    const uint32_t* ivf_postings = nullptr;
    const uint8_t* ivf_mult = nullptr;  // P: tokens of the passage with the posting's code (<= 255, saturating)
    const float* tok_inv = nullptr;     // T: 1 / ||C[code] + residual|| per token (d = 128; TENSOR stage 4)
    // [K][range_n + 1]: offset in c's posting list of its first posting >= r
    // range_w (wave_range_table); the range kernels' run locator
    const uint32_t* range_tab = nullptr;
    uint32_t range_w = 0, range_n = 0;
    float weights[16] = {};
};

// Radix-select scratch (device): one histogram per digit pass plus a grid
// barrier.  Zeroed by the launcher before every select.
struct SelectState {
    unsigned int hist[6][2048];
    unsigned int bar_count;
    unsigned int bar_gen;
    unsigned int bnd_n;                // keys in the boundary bucket (see radix_select_kernel)
    unsigned int pad;
    unsigned long long bnd[1024];      // not zeroed: only [0, bnd_n) is read
};
constexpr size_t kSelectStateZeroBytes = offsetof(SelectState, bnd);

// Histogram select scratch (select_top_hist): a 65536-bin histogram of the
// keys' top 16 bits (built by the kernel that produces the keys; all zero
// between selects — the compaction re-zeroes it) and the control words.
constexpr uint32_t kHistShift = 48;          // bucket = key >> 48: sign, exponent, 7 mantissa bits of the score
constexpr uint32_t kHistZeroBucket = 0x8000u; // bucket of score 0 (the all-masked stage-2 candidates)
struct SelectHist {
    unsigned int hist[65536];
    unsigned int blk[32];       // per 2048-bucket block: the sum of its counts
    unsigned long long above;   // keys in buckets above the boundary bucket
    unsigned long long bcount;  // keys in the boundary bucket
    unsigned long long rem;     // boundary keys still to take
    unsigned int bucket;        // boundary bucket (top 16 key bits)
    unsigned int take_all;      // n <= want
    unsigned long long bn;      // boundary keys written to the side buffer
    unsigned int done;          // CTAs of the select finished (the last one resolves the bucket)
};

constexpr int kScoresPitch = 32;  // S rows padded to 32 floats (128 B)

// Per-query outputs of the (batched) tensor S_cq kernel, query qi < qb.
constexpr uint32_t kMaxScoreBatch = 2;
struct TfOut {
    const float* Q[kMaxScoreBatch];
    float* S[kMaxScoreBatch];
    uint32_t* keep[kMaxScoreBatch];
    uint64_t* partial[kMaxScoreBatch];
    uint32_t* gthr[kMaxScoreBatch];
};

namespace launch {

// True the first time per (call site, current device): kernel attributes
// (e.g. the dynamic shared-memory limit) are per device, so a process that
// drives several GPUs must set them on each.
struct PerDeviceOnce {
    std::atomic<unsigned long long> mask{0};
    bool first() {
        int d = 0;
        cudaGetDevice(&d);
        const unsigned long long bit = 1ull << (d & 63);
        return !(mask.fetch_or(bit) & bit);
    }
};

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while the previous kernel in the stream drains; every kernel
// starts with dev::pdl_wait(), so no data dependence is relaxed.
bool pdl_enabled();  // false when PLAID_NO_PDL is set (ordering experiments)
// Profiling knob (plaid_debug_set_launch_cap): true once this thread has
// issued `cap` launches since reset_launches(), so a search stops after its
// first `cap` kernels (tools/chain_profile.py: marginal cost of each kernel
// inside the PDL chain).  Always false unless the cap is set.
bool pdl_skip();
int64_t set_launch_cap(int64_t cap);  // -1 = no cap; returns the old cap
template <typename... KArgs, typename... Args>
inline void pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    if (pdl_skip()) return;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- stage 1 -----------------------------------------------------------------
// S = C . Q^T (in-order fp32, bit-exact), row max, keep bits (row max >= t_cs),
// and per-warp top-NP keys per query token written to `partial`
// [num_warps][32][np_bucket].  Returns the number of warps used.
uint32_t scores_exact(const IndexView& ix, const float* d_q, uint32_t rows, float t_cs,
                      float* d_scores, float* d_rowmax, uint32_t* d_keep_bits,
                      uint64_t* d_partial, uint32_t np_bucket, cudaStream_t st);
// Max number of warps scores_exact may use (for sizing `partial`).
uint32_t scores_max_warps();
// tcgen05/TMA 3xTF32 variant (gemm_tf32.cu); same outputs, dim == 128 only.
// `cmap` is a CUtensorMap (128 B) made by make_centroid_tensor_map.
bool tensor_scores_supported(const IndexView& ix);
void make_centroid_tensor_map(const IndexView& ix, void* out_map);
// S, keep bits and per-warp top-NP lists (no row max: the pipeline only needs
// the keep bits).  d_gthr: 32 u32 grid-wide per-token bounds, zeroed before
// the launch.  Returns the number of partial lists written.
uint32_t scores_tensor(const void* cmap, const IndexView& ix, const float* d_q, uint32_t rows, float t_cs,
                       float* d_scores, uint32_t* d_keep_bits, uint64_t* d_partial, uint32_t np_bucket,
                       uint32_t* d_gthr, cudaStream_t st);
uint32_t scores_tensor_max_warps();
// Batched variant: qb (<= kMaxScoreBatch) queries share one pass over C
// (B operand = every query's Q_hi and Q_lo, N = 64 qb); per-query outputs as
// above.  nprobe bucket <= 8.  Returns the number of partial lists per query.
uint32_t scores_tensor_batch(const void* cmap, const IndexView& ix, const TfOut& out, uint32_t qb, uint32_t rows,
                             float t_cs, uint32_t np_bucket, cudaStream_t st);
[[noreturn]] void fail_cuda_driver(int code, const char* what);
// Stage 2's kept-centroid list: list (K), counts[0] kept, counts[1] their
// total posting count (both zeroed beforehand).
struct KeepListArgs {
    const uint32_t* keep_bits = nullptr;
    uint32_t* list = nullptr;
    unsigned long long* counts = nullptr;
};
inline uint32_t keep_list_blocks(uint64_t K) {
    const uint64_t kb = ((K + 31) / 32 + 255) / 256;
    return uint32_t(kb ? kb : 1);
}
// topn_merge + postings_to_bitmap in one launch (rows x nprobe CTAs), plus
// the kept-centroid list when `kl` is given (then stage2_masked is called
// with kept_ready).
void topn_postings(const uint64_t* d_partial, uint32_t num_warps, uint32_t np_bucket, uint32_t rows, uint32_t nprobe,
                   const IndexView& ix, uint32_t* d_sel, uint32_t* d_bitmap, const KeepListArgs* kl, cudaStream_t st);
// Merge per-warp partial top-NP lists into sel[rows][nprobe] centroid ids.
void topn_merge(const uint64_t* d_partial, uint32_t num_warps, uint32_t np_bucket, uint32_t rows,
                uint32_t nprobe, uint32_t* d_sel, cudaStream_t st);
// Top-NP per token from a stored S; returns warps used (<= scores_max_warps()).
// d_gthr (optional): 32 u32 grid-wide per-token bounds, zeroed beforehand.
uint32_t topn_from_scores(const float* d_scores, uint64_t K, uint32_t rows, uint64_t* d_partial,
                          uint32_t np_bucket, uint32_t* d_gthr, cudaStream_t st);
void iota(uint32_t* d_out, uint64_t n, cudaStream_t st);
// Keys (S[c][i], c) for one token column i -> keys[K] (generic nprobe path).
void token_keys(const float* d_scores, uint64_t K, uint32_t i, uint64_t* d_keys, cudaStream_t st);
// sel[j] = key_id(keys[j]) for j < n (device count)
void keys_to_ids(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint32_t* d_ids,
                 cudaStream_t st);
// rowmax >= t_cs -> keep bits
void keep_bits_from_rowmax(const float* d_rowmax, uint64_t K, float t_cs, uint32_t* d_keep_bits,
                           cudaStream_t st);

// ---- candidate generation -------------------------------------------------------
void postings_to_bitmap(const IndexView& ix, const uint32_t* d_sel, uint32_t nsel,
                        uint32_t* d_bitmap, cudaStream_t st);
// Bitmap (N bits) -> ascending ids + count.  chunk_counts has bitmap_chunks(N) entries.
uint32_t bitmap_chunks(uint64_t N);
// d_slot_of (optional, N): slot_of[pid] = position of pid in the output.
// Same in one launch; d_status: bitmap_chunks(N) + 1 u64 (chunk flags + ticket counter), zero on entry.
void bitmap_compact_1pass(const uint32_t* d_bitmap, uint64_t N, unsigned long long* d_status, uint32_t* d_out_ids,
                          uint64_t* d_out_n, uint32_t* d_slot_of, cudaStream_t st);
void bitmap_compact(const uint32_t* d_bitmap, uint64_t N, uint32_t* d_chunk_counts,
                    uint32_t* d_out_ids, uint64_t* d_out_n, uint32_t* d_slot_of, cudaStream_t st);

// ---- centroid interaction (stages 2 and 3) -----------------------------------------
// Candidates are either ids (d_ids) or keys (d_keys, id in the low word).
// Writes keys (score, id) and optionally raw scores; adds used rows to *d_rows.
// d_owners (optional, masked only): N-bit set of passages owning a kept token
// (kept_owners); candidates outside it are scored 0 without reading codes.
void centroid_interaction(const IndexView& ix, const float* d_scores, uint32_t rows,
                          const uint32_t* d_ids, const uint64_t* d_keys, const uint64_t* d_n,
                          uint64_t nmax, const uint32_t* d_keep_bits, const uint32_t* d_owners,
                          uint64_t* d_out_keys, float* d_out_scores, unsigned long long* d_rows,
                          cudaStream_t st, uint32_t* d_out_len = nullptr, uint64_t* d_out_off = nullptr);
// owners |= postings(c) for every kept centroid c (owners zeroed by the caller).
void kept_owners(const IndexView& ix, const uint32_t* d_keep_bits, uint32_t* d_owners, cudaStream_t st);
// Stage 2 over C1 (ids d_c1 ascending, count *d_n1 <= nmax, membership
// bitmap d_cand_bits): keys for every candidate, from the kept centroids'
// posting lists (interaction.cu).  Scratch: d_used_bits (nmax bits, zeroed),
// d_counts2 (2 zeroed counters), d_kept_list (K), d_slot_of (N), d_acc
// (nmax x 32, all zero between calls).
void stage2_masked(const IndexView& ix, const float* d_scores, uint32_t rows, const uint32_t* d_c1,
                   const uint64_t* d_n1, uint64_t nmax, const uint32_t* d_keep_bits, const uint32_t* d_cand_bits,
                   uint32_t* d_used_bits, uint32_t* d_kept_list, const uint32_t* d_slot_of, uint32_t* d_acc,
                   unsigned long long* d_counts2, uint64_t* d_out_keys, unsigned long long* d_rows,
                   SelectHist* d_hist, bool kept_ready, cudaStream_t st);

// Candidate generation + stage 2 in one launch, a CTA per pid range
// (range_stage2.cu): from the probed centroids sel[nsel] and the kept list
// (topn_postings' kl outputs), stage-2 keys of every C1 member into
// d_keys[0..*d_n1) (order unspecified), the select histogram, the
// stage1_candidates / stage2_rows_gathered counters.  Needs ix.range_tab.
bool range_stage2_ok(const IndexView& ix, uint32_t rows, uint64_t nsel);
// d_ukeys / d_nu (optional, *d_nu zero on entry): the keys of the candidates
// owning a kept token again, compact — every positive stage-2 key is there.
void range_stage2(const IndexView& ix, const float* d_scores, uint32_t rows, const uint32_t* d_sel, uint32_t nsel,
                  const uint32_t* d_keep_bits, const uint32_t* d_kept, const unsigned long long* d_kept_counts,
                  uint64_t* d_keys, uint64_t* d_n1, unsigned long long* d_rows, SelectHist* d_hist,
                  uint64_t* d_ukeys, uint64_t* d_nu, cudaStream_t st);

// ---- selection -----------------------------------------------------------------------
// Top `want` of keys[0..*d_n) (largest first).  Result: d_out_keys unsorted
// (count min(want, n) in *d_out_n).  Uses radix select over 64-bit keys.
void select_top_large(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want,
                      SelectState* d_state, uint64_t* d_out_keys, uint64_t* d_out_n,
                      cudaStream_t st);
// Same result as select_top_large without grid barriers, from the key
// histogram d_st->hist built by the keys' producer (range_stage2 /
// stage2_finalize / ci_all), in ONE launch: every CTA finds the boundary
// bucket and compacts its share (keys above it -> out, bucket keys ->
// d_bkeys, capacity nmax); the last CTA to finish (ticket d_st->done)
// resolves the bucket by a shared-memory radix select (global memory past
// 16384 keys) and re-zeroes the histogram.  *d_out_n must be zero on entry.  d_ukeys / d_nu (optional): the
// keys with a positive-capable score (stage 2: candidates owning a kept
// token), scanned instead of all keys when the boundary lies above score 0.
void select_top_hist(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want, SelectHist* d_st,
                     uint64_t* d_bkeys, uint64_t* d_out_keys, uint64_t* d_out_n, cudaStream_t st,
                     const uint64_t* d_ukeys = nullptr, const uint64_t* d_nu = nullptr);
// Sort keys[0..*d_n) descending (n <= nmax) and emit the first min(want, n):
// out_keys (optional), out_ids/out_scores (optional, ids offset by id_base),
// out_n (optional).  nmax <= kSmallSortMax uses one CTA; larger uses a
// global bitonic sort in `d_tmp` (capacity next_pow2(nmax)).
constexpr uint64_t kSmallSortMax = 8192;
void sort_top(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want,
              uint64_t* d_out_keys, uint32_t* d_out_ids, float* d_out_scores, uint64_t* d_out_n,
              uint32_t id_base, uint64_t* d_tmp, cudaStream_t st);
uint64_t sort_tmp_capacity(uint64_t nmax);
// Stage 4's finalize (per-finalist sum of the running maxima `run`) fused with
// the final top-k rank sort: one launch instead of finalize + sort_top.  For
// kFinalRankMin <= nmax <= kSmallSortMax.  Leaves `run` zero like
// finalize_kernel; *d_ticket must be 0 at launch.
constexpr uint64_t kFinalRankMin = 256;
void finalize_rank(const uint32_t* d_ids, const uint64_t* d_fkeys, const uint64_t* d_n, uint64_t nmax, uint32_t rows,
                   uint32_t* d_run, uint64_t want, uint32_t* d_out_ids, float* d_out_scores, uint64_t* d_out_n,
                   uint32_t id_base, unsigned int* d_ticket, cudaStream_t st);
// Stage 4's finalist scan outputs (RankScratch pref / fin_base / tokens) and
// the index arrays it reads.
struct FinalistScanArgs {
    const uint32_t* doclens = nullptr;
    const uint64_t* offsets = nullptr;
    uint32_t* pref = nullptr;
    uint64_t* fin_base = nullptr;
    uint64_t* tokens = nullptr;
    uint32_t* run_p0 = nullptr;  // finalist of every 32nd stream position (TENSOR stage 4)
    // optional: (doclen, offset) of every select input (centroid_interaction's
    // out_len / out_off), so the scan reads them from shared memory instead of
    // two dependent L2 round trips per finalist
    const uint32_t* cand_len = nullptr;
    const uint64_t* cand_off = nullptr;
};
// The top-`want` SET of keys[0..*d_n) (unordered), nmax <= kSmallSortMax, one
// CTA (shared-memory radix select); *d_out_n = min(n, want).  With `fs`, the
// same CTA then runs stage 4's finalist scan over the set (rank_exact is
// then called with RankScratch::prescanned).
void select_set(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want, uint64_t* d_out_keys,
                uint64_t* d_out_n, const FinalistScanArgs* fs, cudaStream_t st);

// Global-exact shard exchange (select.cu): export keys[0..*d_n) in global
// form (ids + base) into a zero-padded row of `stride`; then, from the
// all-gathered rows of every shard (total keys), keep in place only the local
// keys at or above the global want-th largest key (*d_n updated).
void export_keys(const uint64_t* d_keys, const uint64_t* d_n, uint64_t stride, uint32_t base, uint64_t* d_out,
                 cudaStream_t st);
// All-gather as one kernel on the calling stream's device: row g of d_dst
// (`words` u64 each) <- src.p[g], read through peer access when the shards
// live on other GPUs.
constexpr uint32_t kMaxShards = 16;
struct PeerRows {
    const uint64_t* p[kMaxShards];
};
void gather_rows(const PeerRows& src, uint32_t shards, uint64_t words, uint64_t* d_dst, cudaStream_t st);
// Batch merge of shard top-k lists ([shards][B][k] pids / scores, counts
// [shards][B]) into [B][k] + out_n[B]; shards * k <= 25600.
void merge_batch(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts, uint32_t shards, uint32_t B,
                 uint32_t k, uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n, cudaStream_t st);
void threshold_filter(const uint64_t* d_gathered, uint64_t total, uint64_t want, uint64_t* d_keys, uint64_t* d_n,
                      uint32_t base, cudaStream_t st);

// ---- stage 4 ----------------------------------------------------------------------
// Decompress + exact MaxSim per candidate (ids from keys or ids); writes keys.
// With d = 128 and a finalist list that fits `scratch` (rank128.cu: the
// packed token-stream path), otherwise one fused kernel per finalist.
struct RankScratch {
    uint32_t* pref = nullptr;     // pass_cap + 1: stream offset of each finalist
    uint32_t* run = nullptr;      // pass_cap x 32 running maxima; all zero between searches
    uint64_t* fin_base = nullptr; // pass_cap: index token of stream position g is fin_base[p] + g
    uint64_t* tokens = nullptr;   // 1 counter: stage-4 stream length (trace)
    uint64_t pass_cap = 0;
    bool prescanned = false;      // pref / fin_base / tokens already written (select_set)
    const float* tensor_S = nullptr;  // TENSOR mode: this query's S_cq table -> stage4_tensor_kernel
    uint32_t* run_p0 = nullptr;       // TENSOR mode: finalist of every 32nd stream position (scan output)
    const void* qimg = nullptr;       // TENSOR mode: the query's bf16 B-operand image (query_prologue)
    // set: rank_stream128 ends with finalize_rank into these (top-k ids and
    // scores) instead of finalize_kernel's keys; `run` must arrive zeroed
    struct Final {
        uint64_t want = 0;
        uint32_t* ids = nullptr;
        float* scores = nullptr;
        uint64_t* n = nullptr;
        uint32_t base = 0;
        unsigned int* ticket = nullptr;  // zero at launch (a per-query counter)
    };
    const Final* final_out = nullptr;
    // TENSOR mode: stage 4 as a warp per finalist on mma.sync (s4_mma.cuh)
    // writing the finalists' keys, instead of stage4_tensor_kernel's tiles
    bool warp_s4 = false;
};
// Bytes of the stage-4 tensor kernel's B-operand image of a query (built by
// query_prologue when given a destination).
constexpr uint32_t kQImgBytes = 32 * 1024;
// ... followed by the query's mma.sync B fragments (s4_mma.cuh layout,
// [k-step][n-tile][hi, lo][lane] uint2) for stage4_warp_kernel
constexpr uint32_t kQFragImgBytes = 8 * 4 * 2 * 32 * 8;
// inv_t = 1 / ||C[code_t] + r_t|| for every index token (d = 128), the
// reference's arithmetic (residual_codec.cpp:113-130); index-load time.
void token_inv_norms(const IndexView& ix, float* d_out, cudaStream_t st);
constexpr uint64_t kStreamMaxPassages = 16384;
void rank_exact(const IndexView& ix, const float* d_q, uint32_t rows, const uint32_t* d_ids,
                const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t* d_out_keys,
                const RankScratch* scratch, cudaStream_t st);
// Whether rank_exact takes the streamed path (rank_stream128) for this shape.
bool rank_stream128_ok(const IndexView& ix, uint32_t rows, uint64_t nmax, const RankScratch& s);
bool rank_stream128(const IndexView& ix, const float* d_q, uint32_t rows, const uint32_t* d_ids,
                    const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t* d_out_keys,
                    const RankScratch& s, cudaStream_t st);

// ---- throughput mode: waves of queries (wave_scores.cu, wave_worker.cu) ------------
// S_cq of a wave, 4 queries per pass over C (tcgen05, 3xTF32): S rows
// [nq][s_stride], keep bits [nq][keep_stride], partial top-NP lists
// [nq][partial_stride] as [wave_scores_lists()][32][np_bucket] (key 0 = empty).  Q: [nq][rows][128].
void make_wave_tensor_map(const IndexView& ix, void* out_map);
uint32_t wave_scores_lists(const IndexView& ix);
uint32_t wave_scores(const void* cmap, const IndexView& ix, const float* d_q, uint32_t nq, uint32_t rows, float t_cs,
                     uint32_t np_bucket, float* d_S, uint64_t s_stride, uint32_t* d_keep, uint64_t keep_stride,
                     uint64_t* d_partial, uint64_t partial_stride, cudaStream_t st);
constexpr uint32_t kWaveSortCap = 2048;     // max finalists (stage3_width) of the wave worker
constexpr uint32_t kWaveRangeIds = 65536;   // pid range of the worker's shared-memory member bitmap
constexpr uint32_t kRangeIdsMax = 131072;   // widest pid range of range_stage2 (its member bitmap)
// range_stage2's pid range width for N passages: about one range per SM
// (power of two, 1024 .. kRangeIdsMax ids)
inline uint32_t range_width_for(uint64_t N, uint32_t sms) {
    uint64_t w = 1024;
    while (w < kRangeIdsMax && w * sms < N) w <<= 1;
    return uint32_t(w);
}
// Index-side table of the wave worker: for centroid c and pid range r (ids
// [r W, (r+1) W)), the offset in c's posting list of its first posting >= r W;
// [K][R + 1] u32 with R = ceil(N / W).
void wave_range_table(const IndexView& ix, uint32_t W, uint32_t R, uint32_t* d_tab, cudaStream_t st);
// Per-wave buffers of the worker: slot q (= query q of the wave) owns c1 /
// keys [c1cap], side [3 c1cap], acc [ndocs x 32] (zero between queries),
// sel [sel_stride >= ndocs + n3].
struct WaveArgs {
    const float* Q = nullptr;
    uint32_t rows = 0, nprobe = 0, ndocs = 0, n3 = 0, k = 0, nlists = 0, pid_base = 0, validate = 0;
    uint32_t s4_tensor = 0;  // stage 4 as (S + R Q^T) * inv on mma.sync (TENSOR mode; else exact)
    const float* S = nullptr;
    uint64_t s_stride = 0;
    const uint32_t* keep = nullptr;
    uint64_t keep_stride = 0;
    const uint64_t* partial = nullptr;
    uint64_t partial_stride = 0;
    const uint32_t* range_tab = nullptr;
    uint32_t range_w = 0, range_n = 0;
    uint32_t* c1 = nullptr;
    uint32_t* acc = nullptr;
    uint64_t* keys = nullptr;
    uint64_t* side = nullptr;
    uint64_t c1cap = 0;
    uint64_t* sel = nullptr;
    uint64_t sel_stride = 0;
    uint32_t* out_pids = nullptr;
    float* out_scores = nullptr;
    uint64_t* out_n = nullptr;
    uint64_t* counters = nullptr;  // optional [nq][4]: stage1, stage2_out, stage3_out, final_out
    int* status = nullptr;
    unsigned long long* trace = nullptr;  // optional [nq][16] phase timestamps (globaltimer)
};
void wave_worker(const IndexView& ix, const WaveArgs& a, uint32_t nq, uint32_t np_stride, cudaStream_t st);
uint32_t wave_worker_ctas_per_sm(uint32_t nbits);  // resident worker CTAs per SM (occupancy)

// ---- misc ---------------------------------------------------------------------------
// Device-side query validation (types.cpp:61-72, status 0 or NotNormalized+1)
// query validation (when d_q != nullptr) + zero nwords u32 at d_zero and nwords2
// at d_zero2 (multiples of 4 words, 16-byte aligned): one launch.
// d_qimg (optional, kQImgBytes): also build the stage-4 tensor kernel's
// B-operand image of the query at d_qsrc (rows x 128).
// d_qcopy (optional): first copy the rows x dim query from d_qsrc (e.g. a
// mapped pinned host buffer) to d_qcopy.
void query_prologue(const float* d_q, uint32_t rows, uint32_t dim, int* d_status, uint32_t* d_zero, uint64_t nwords,
                    uint32_t* d_zero2, uint64_t nwords2, cudaStream_t st, const float* d_qsrc = nullptr,
                    void* d_qimg = nullptr, float* d_qcopy = nullptr);
// One CTA: words u32 (multiple of 4) d_src -> mapped host h_dst, then
// *h_flag = ++*d_seq (system-scope fences between).
void publish(const uint32_t* d_src, uint32_t* h_dst_mapped, uint64_t words, unsigned int* d_seq,
             unsigned int* h_flag_mapped, cudaStream_t st);
// Stage counters: min() bookkeeping done on device.
void copy_count(const uint64_t* src, uint64_t* dst, uint64_t cap, cudaStream_t st);
// Merge G shard top-k lists into the global top-k.
// Shard g's list: pids[g * stride + j], scores[g * stride + j] for j <
// min(per, counts[g * count_stride]) (count_stride 1 = a separate count array).
void merge_topk(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts,
                uint64_t shards, uint64_t stride, uint64_t count_stride, uint64_t per, uint64_t k,
                uint64_t* d_tmp_keys, uint64_t* d_tmp_n, uint32_t* d_out_pids, float* d_out_scores,
                uint64_t* d_out_n, uint64_t* d_sort_tmp, cudaStream_t st);
// Build keys from (ids, scores) arrays (select_top entry point).
void make_keys(const uint32_t* d_ids, const float* d_scores, uint64_t n, uint64_t* d_keys,
               cudaStream_t st);

// ---- codec / maxsim entry points -------------------------------------------------
void unpack_via_lut(const uint8_t* d_packed, uint64_t n, uint32_t nbits, uint8_t* d_out,
                    cudaStream_t st);
void reconstruct(const IndexView& ix, const uint32_t* d_codes, uint64_t n,
                 const uint8_t* d_residuals, float* d_out, cudaStream_t st);
void maxsim_packed(const float* d_scores, uint32_t nq, const uint64_t* d_offsets, uint64_t np,
                   float* d_out, cudaStream_t st);
void maxsim_embeddings(const float* d_q, uint32_t rows, uint32_t dim, const float* d_emb,
                       const uint64_t* d_offsets, uint64_t np, float* d_out, cudaStream_t st);

// Number of kernel launches issued by this thread since the last reset.
uint64_t launches();
void reset_launches();
void count_launch();

}  // namespace launch
}  // namespace plaid
