// engine.hpp — C++ host side of the B200 PLAID searcher.
//
// DeviceIndex mirrors lir::CompressedIndex (index.hpp:60-85) in HBM; Searcher
// owns one stream and all per-query scratch, pre-sized from (K, N) so a search
// never allocates, and enqueues the four stages of lir::search
// (pipeline.cpp:232-283) as a fixed launch sequence.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/plaid.h"
#include "kernels.cuh"

namespace plaid {

class Error : public std::runtime_error {
public:
    Error(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
    int status() const noexcept { return status_; }

private:
    int status_;
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

void cuda_check(cudaError_t e, const char* what);
#define PLAID_CUDA(x) ::plaid::cuda_check((x), #x)

// Makes `dev` current for the scope.
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) PLAID_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

// Host-side validation mirroring types.cpp / index.cpp.
void validate_query_host(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim);
void validate_params_host(const plaid_params& p, uint64_t num_centroids);
void default_params_for_k(uint64_t k, plaid_params* out);
uint64_t stage3_width(const plaid_params& p);
void validate_index_host(const plaid_index_desc& d);

// The synthetic index recipe of SURVEY.md §8d (plaid_index_synth).
struct SynthSpec {
    uint64_t num_passages = 0, num_centroids = 0, pid_base = 0, seed = 0;
    uint32_t dim = 128, nbits = 2, mean_len = 64, spread = 16;
    double repeat = 0.28;
};

class DeviceIndex {
public:
    DeviceIndex(const plaid_index_desc& d, int device, uint64_t pid_base);
    // Generated in HBM (synth_device.cu): passages [pid_base, pid_base + N)
    // of the synthetic corpus, local IVF, global ids in results.
    DeviceIndex(const SynthSpec& spec, int device);
    void synth_queries(uint64_t nq, uint32_t qlen, double noise, uint64_t seed, float* out_host) const;
    void export_host(float* centroids, uint32_t* codes, uint8_t* residuals, uint32_t* doclens, uint64_t* ivf_offsets,
                     uint32_t* ivf_postings, float* cutoffs, float* weights) const;
    ~DeviceIndex();
    DeviceIndex(const DeviceIndex&) = delete;
    DeviceIndex& operator=(const DeviceIndex&) = delete;

    const IndexView& view() const { return view_; }
    int device() const { return device_; }
    uint64_t pid_base() const { return pid_base_; }
    uint32_t max_doclen() const { return max_doclen_; }
    uint64_t bytes() const { return bytes_; }
    const float* cutoffs() const { return cutoffs_; }
    const std::vector<uint32_t>& host_doclens() const { return h_doclens_; }
    // Downloads the device arrays and re-checks validate_index's invariants.
    void validate_device();
    // Upper bound on |C1| for a query probing nprobe centroids per token:
    // at most 32 * nprobe distinct lists, so at most the sum of the 32 *
    // nprobe longest list lengths (and at most N).  Sizes the stage-2
    // accumulators by the query's reach instead of the corpus.
    uint64_t candidate_bound(uint64_t nprobe) const;

private:
    template <typename T>
    T* upload(const T* src, uint64_t count);
    int device_;
    uint64_t pid_base_;
    IndexView view_;
    uint32_t max_doclen_ = 0;
    uint64_t bytes_ = 0;
    float cutoffs_[16] = {};
    std::vector<void*> allocs_;
    std::vector<uint32_t> h_doclens_;
    std::vector<uint64_t> longest_prefix_;  // [K + 1]: sums of the j longest list lengths
    void set_list_bounds(const uint64_t* ivf_offsets_host);
    void build_range_table(cudaStream_t st);
};

// Host-side pinned/device buffer helper.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    uint64_t n = 0;
    void ensure(uint64_t count);
    void release();
    ~DevBuf() { release(); }
};

struct SearchCounts;  // device-side trace counters

class Searcher {
public:
    Searcher(DeviceIndex* index, int device, const plaid_searcher_config& cfg);
    ~Searcher();

    // Host path (lir::search): validates, uploads Q, runs, downloads.
    void search(const float* q, uint64_t rows, uint64_t dim, const plaid_params& p,
                uint32_t* out_pids, float* out_scores, uint64_t* out_n, plaid_trace* trace);
    // Device path: enqueue only.
    void search_device(const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim,
                       const plaid_params& p, uint32_t* d_pids, float* d_scores, uint64_t* d_n,
                       cudaStream_t st);
    // Global-exact sharded search: phases separated by the caller's all-gathers.
    void shard_phase1(const float* d_q, uint64_t rows, uint64_t dim, const plaid_params& p, uint64_t* d_x2,
                      uint64_t stride2, cudaStream_t st);
    void shard_phase2(const uint64_t* d_g2, uint64_t shards, uint64_t* d_x3, uint64_t stride3, cudaStream_t st);
    void shard_phase3(const uint64_t* d_g3, uint64_t shards, uint32_t* d_pids, float* d_scores, uint64_t* d_n,
                      cudaStream_t st);
    void trace_counters_device(uint64_t* d_out, cudaStream_t st);
    // Batched S_cq (BatchSearcher): prologue, this lane's S_cq outputs, the rest.
    bool batch_scores_ok(const plaid_params& p, uint64_t rows, uint64_t dim) const;
    void batch_prepare(const float* d_q, uint64_t rows, uint64_t dim, const plaid_params& p, cudaStream_t st);
    void batch_targets(TfOut& out, uint32_t qi, const float* d_q);
    void batch_finish(const float* d_q, uint32_t rows, const plaid_params& p, uint32_t warps, uint32_t* d_pids,
                      float* d_scores, uint64_t* d_n, cudaStream_t st);
    const void* tensor_map() const { return tmap_; }
    void sync();
    uint64_t last_launches() const { return last_launches_; }
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }
    void phase_ms(double* out);

    // Per-stage entry points (host buffers).
    void compute_centroid_scores(const float* q, uint64_t rows, uint64_t dim, float* scores,
                                 float* row_max);
    void generate_candidates(const float* scores, uint64_t rows, uint64_t nprobe, uint32_t* out_ids,
                             uint64_t* out_n);
    void centroid_interaction(const float* scores, uint64_t rows, const uint32_t* cand, uint64_t n,
                              const uint8_t* mask, float* out_scores, uint64_t* rows_gathered);
    void select_top(const uint32_t* ids, const float* scores, uint64_t n, uint64_t keep,
                    uint32_t* out_ids, float* out_scores, uint64_t* out_n);
    void rank_final(const float* q, uint64_t rows, const uint32_t* cand, uint64_t n, uint64_t k,
                    uint32_t* out_ids, float* out_scores, uint64_t* out_n);
    void reconstruct(const uint32_t* codes, uint64_t n, const uint8_t* residuals, float* out);
    void unpack(const uint8_t* packed, uint64_t n, uint32_t nbits, uint8_t* out);
    void maxsim_packed(const float* scores, uint64_t nq, const uint64_t* offsets, uint64_t np,
                       float* out);
    void maxsim_embeddings(const float* q, uint64_t rows, uint64_t dim, const float* emb,
                           const uint64_t* offsets, uint64_t np, float* out);
    void merge_topk(const uint32_t* pids, const float* scores, const uint64_t* counts,
                    uint64_t shards, uint64_t stride, uint64_t k, uint32_t* out_pids,
                    float* out_scores, uint64_t* out_n);
    void merge_topk_device(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts,
                           uint64_t shards, uint64_t stride, uint64_t k, uint32_t* d_out_pids,
                           float* d_out_scores, uint64_t* d_out_n, cudaStream_t st);
    void merge_topk_rows_device(const uint32_t* d_rows, uint64_t shards, uint64_t k, uint32_t* d_out_pids,
                                float* d_out_scores, uint64_t* d_out_n, cudaStream_t st);

private:
    void require_index() const;
    // Enqueue one query whose rows already sit at d_q; results go to the
    // given device buffers (pids are global: local + pid_base).
    void enqueue(const float* d_q, uint32_t rows, const plaid_params& p, uint32_t* d_pids,
                 float* d_scores, uint64_t* d_n, cudaStream_t st, bool times, bool validate);
    void enqueue_front(const float* d_q, uint32_t rows, const plaid_params& p, cudaStream_t st, bool times,
                       bool validate);
    void front_after_scores(uint32_t rows, const plaid_params& p, uint32_t warps, cudaStream_t st, bool times);
    // candidates + stage 2 through range_stage2 (no bitmaps to clear)
    bool range_path(uint32_t rows, const plaid_params& p) const;
    // stage 4 ends in one finalize_rank launch (else finalize_kernel + sort_top)
    bool final_fused_ok(uint32_t rows, const plaid_params& p) const;
    void enqueue_stage3(const plaid_params& p, cudaStream_t st, bool times, bool fuse_scan);
    void enqueue_back(const float* d_q, uint32_t rows, const plaid_params& p, uint32_t* d_pids, float* d_scores,
                      uint64_t* d_n, cudaStream_t st, bool times);
    void ensure_param_buffers(const plaid_params& p);
    void ensure_param_buffers_impl(const plaid_params& p);
    void ensure_result_block(uint64_t k);
    void record(int slot, cudaStream_t st, bool times);

    DeviceIndex* index_;
    int device_;
    plaid_searcher_config cfg_;
    cudaStream_t stream_ = nullptr;
    uint64_t last_launches_ = 0;
    // launches of the shard phases of the pending query, counted per call so
    // several searchers' phases may interleave on one host thread
    uint64_t phase_launches_ = 0;
    // captured host-path graphs (plaid_searcher_config.use_graphs)
    struct GraphKey {
        uint64_t rows, k, nprobe, ndocs;
        int32_t disable_filter;
        uint32_t t_cs_bits;
        bool operator==(const GraphKey& o) const {
            return rows == o.rows && k == o.k && nprobe == o.nprobe && ndocs == o.ndocs &&
                   disable_filter == o.disable_filter && t_cs_bits == o.t_cs_bits;
        }
    };
    struct GraphEntry {
        GraphKey key;
        uint64_t gen;
        cudaGraphExec_t exec;
        uint64_t launches;
    };
    std::vector<GraphEntry> graphs_;
    // sharded-search state between shard_phase calls
    plaid_params pending_{};
    const float* pending_q_ = nullptr;
    uint32_t pending_rows_ = 0;
    uint64_t pending_stride2_ = 0, pending_stride3_ = 0;
    int phase_ = 0;

    // scratch
    DevBuf<float> q_, scores_, rowmax_;
    DevBuf<uint32_t> keep_, sel_, chunk_counts_, c1_, ids_tmp_, pref_, run_, slot_of_, kept_list_, acc2_;
    DevBuf<uint32_t> run_p0_, qimg_;  // TENSOR stage 4: finalist per 32 stream tokens, query B-operand image
    // result block [32 u64 counters | k pids | k scores] (ensure_result_block)
    DevBuf<uint32_t> res_;
    uint64_t res_k_ = 0;
    uint32_t* out_pids_p_ = nullptr;
    float* out_scores_p_ = nullptr;
    uint32_t* h_res_ = nullptr;
    launch::RankScratch rank_scratch_;
    bool scan_fused_ = false;  // stage 3's select ran stage 4's finalist scan
    DevBuf<uint64_t> partial_, tok_keys_, keys2_, ukeys_, sel2_, keys3_, sel3_, keys4_, sel4_, sort_tmp_, fin_base_, bkeys_,
        tmp_keys_, kconst_;
    DevBuf<uint32_t> cand_len_;  // stage-3 candidates' doclens, carried to the finalist scan
    DevBuf<uint64_t> cand_off_;  // ... and their token offsets
    // zero_ = [16 u64 counters | candidate bitmap (N bits) | kept-owner bitmap
    // (N bits)], cleared by a single memset per query.
    DevBuf<uint32_t> zero_;
    unsigned long long* compact_status_ = nullptr;  // inside zero_ (bitmap_compact_1pass)
    template <typename T>
    struct View {
        T* p = nullptr;
    };
    View<uint64_t> counters_;
    View<uint32_t> bitmap_;
    DevBuf<unsigned char> bytes_tmp_;
    DevBuf<SelectState> sel_state_;
    DevBuf<SelectHist> sel_hist_;
    DevBuf<int> status_;
    // pinned staging (mapped: read / written by kernels directly on the host path)
    float* h_q_ = nullptr;
    const float* host_q_ = nullptr;      // set while the host path enqueues
    unsigned int* h_flag_ = nullptr;     // publish flag (pinned)
    unsigned int pub_seq_host_ = 0;
    DevBuf<uint32_t> pub_seq_;           // publish sequence on the device
    void wait_published();
    cudaEvent_t ev_[8] = {};
    uint64_t npartial_warps_ = 0;
    bool tensor_ = false;                   // tcgen05 S_cq path active
    alignas(64) unsigned char tmap_[128];   // CUtensorMap over the centroids
    // S_cq + row max + keep bits + per-warp top lists, in the configured mode
    uint32_t launch_scores(const float* d_q, uint32_t rows, float t_cs, uint32_t npb, cudaStream_t st);
};

// Throughput mode, wave engine: a batch runs in waves of up to `slots`
// queries; per wave ONE S_cq pass (TENSOR: wave_scores, four queries per
// pass over C; EXACT: the exact kernel per query) and ONE worker launch with
// a CTA per query for stages 1b-4 (wave_worker.cu).  Scratch is per slot,
// sized from the index and the params (throughput mode).
class WavePipeline {
public:
    WavePipeline(DeviceIndex* index, int device, bool tensor);
    ~WavePipeline();
    WavePipeline(const WavePipeline&) = delete;
    WavePipeline& operator=(const WavePipeline&) = delete;
    bool supports(const plaid_params& p, uint64_t rows, uint64_t dim) const;
    // d_q [nq][rows][dim]; outputs [nq][k] + d_n[nq] (global ids); the
    // per-query counters [stage1, stage2_out, stage3_out, final_out] stay in
    // the pipeline (counters()).  validate: device-side query norm check.
    void run(const float* d_q, uint64_t nq, uint32_t rows, const plaid_params& p, uint32_t* d_pids, float* d_scores,
             uint64_t* d_n, bool validate, cudaStream_t st);
    void counters(uint64_t* out_host, uint64_t nq);
    // S_cq (K x 32, row per centroid) the last wave computed for its query j
    void copy_scores(uint64_t j, float* out_host);
    // phase timeline of the last batch ([nq][16] globaltimer stamps; needs PLAID_WAVE_TRACE=1)
    void trace(uint64_t* out_host, uint64_t nq);
    void check_status();
    uint64_t last_launches() const { return last_launches_; }
    uint32_t slots() const { return slots_; }

private:
    void ensure(uint64_t nq, const plaid_params& p);
    DeviceIndex* index_;
    int device_;
    bool tensor_;
    alignas(64) unsigned char tmap_[128];
    uint32_t slots_ = 0;
    uint64_t c1cap_ = 0, sel_stride_ = 0, partial_stride_ = 0, keep_stride_ = 0, nd_cap_ = 0, s_stride_ = 0;
    uint64_t last_launches_ = 0;
    DevBuf<float> S_, rowmax_;
    DevBuf<uint32_t> keep_, c1_, acc_, range_tab_;  // range_tab_: 64K-id table when the index's differs
    const uint32_t* range_tab_p_ = nullptr;
    DevBuf<uint64_t> partial_, keys_, side_, sel_, counters_, trace_;
    DevBuf<int> status_;
    bool tracing_ = false;
};

// Throughput mode (BASELINE configs[2]: batched queries): L lanes, each a
// full Searcher with its own stream and scratch over the shared index.
// Query j runs on lane j mod L, so the latency-bound stage kernels of
// different queries overlap on the GPU; a batch forks from and joins back
// to the caller's stream with events.
class BatchSearcher {
public:
    BatchSearcher(DeviceIndex* index, int device, const plaid_searcher_config& cfg, uint32_t lanes);
    ~BatchSearcher();
    uint32_t lanes() const { return uint32_t(lanes_.size()); }
    // Host buffers: Q [nq][rows][dim], outputs [nq][k] + counts [nq].  Each
    // query is validated host-side first (types.cpp:61-99 order).
    void search(const float* q, uint64_t nq, uint64_t rows, uint64_t dim, const plaid_params& p,
                uint32_t* out_pids, float* out_scores, uint64_t* out_n);
    // Device buffers, enqueued on `st` (0 = lane 0's stream); not synchronised.
    void search_device(const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim, const plaid_params& p,
                       uint32_t* d_pids, float* d_scores, uint64_t* d_n, cudaStream_t st);
    void sync();
    uint64_t last_launches() const { return last_launches_; }
    // Which engine ran the last batch (1 = waves, 0 = lanes) and its per-query
    // counters [nq][stage1, stage2_out, stage3_out, final_out] (waves only).
    bool last_was_wave() const { return last_wave_; }
    void wave_counters(uint64_t* out_host, uint64_t nq);
    void wave_scores(uint64_t j, float* out_host);
    void wave_trace(uint64_t* out_host, uint64_t nq);
    uint32_t wave_slots() const { return wave_ ? wave_->slots() : 0; }

private:
    void search_device_impl(const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim, const plaid_params& p,
                            uint32_t* d_pids, float* d_scores, uint64_t* d_n, cudaStream_t st, bool validate);
    DeviceIndex* index_;
    int device_;
    std::unique_ptr<WavePipeline> wave_;  // null when the config asks for lanes only
    bool last_wave_ = false;
    std::vector<std::unique_ptr<Searcher>> lanes_;
    std::vector<cudaStream_t> streams_;
    std::vector<cudaEvent_t> joins_, ready_, sdone_;
    cudaEvent_t fork_ = nullptr;
    cudaStream_t sstream_ = nullptr;  // batched S_cq launches
    uint64_t last_launches_ = 0;
    DevBuf<float> q_;
    DevBuf<uint32_t> pids_;
    DevBuf<float> scores_;
    DevBuf<uint64_t> n_;
    float* h_q_ = nullptr;
    uint32_t* h_pids_ = nullptr;
    float* h_scores_ = nullptr;
    uint64_t* h_n_ = nullptr;
    uint64_t hq_cap_ = 0, ho_cap_ = 0;
};

// Single-process passage-sharded search over G shard indexes
// on one or several GPUs: one Searcher per shard (on the shard's device, its
// own stream), the global-exact protocol of Searcher::shard_phase{1,2,3} (or
// shard-local: whole search per shard, merge only), every exchange an
// on-device all-gather (launch::gather_rows) that reads the other shards'
// exported rows through NVLink peer access, ordered by cross-device events;
// the per-shard top-k rows are gathered and merged on shard 0's device.
// Equals lir::search over the unsharded index (global-exact).
class ShardedSearcher {
public:
    enum Mode { kGlobalExact = 0, kShardLocal = 1 };
    ShardedSearcher(const std::vector<DeviceIndex*>& shards, const plaid_searcher_config& cfg, int mode);
    ~ShardedSearcher();
    void search(const float* q, uint64_t rows, uint64_t dim, const plaid_params& p, uint32_t* out_pids,
                float* out_scores, uint64_t* out_n, plaid_trace* trace);
    uint64_t last_launches() const { return last_launches_; }

private:
    struct Shard {
        DeviceIndex* ix = nullptr;
        std::unique_ptr<Searcher> s;
        int dev = 0;
        cudaStream_t st = nullptr;
        cudaEvent_t ev[3] = {};
        DevBuf<float> q;
        DevBuf<uint64_t> x2, g2, x3, g3, rows, cnt;
        uint64_t* h_cnt = nullptr;  // pinned: this shard's 6 trace counters
    };
    void gather(Shard& dst, int which, uint64_t words, uint64_t* out);
    std::vector<Shard> sh_;
    int mode_;
    uint64_t N_ = 0, dim_ = 0, K_ = 0;
    DevBuf<uint64_t> grows_;   // shard 0: gathered result rows
    DevBuf<uint32_t> out_;     // shard 0: merged [k pids | k scores | n]
    uint32_t* h_out_ = nullptr;
    uint64_t h_out_k_ = 0;
    float* h_q_ = nullptr;
    uint64_t last_launches_ = 0;
};

}  // namespace plaid
