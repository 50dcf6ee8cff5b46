// plaid_lir.hpp — header-only C++ binding of libplaid (plaid.h) for code
// written against the reference searcher `lir` (/root/reference/proj/include).
//
// This is the reference-side binding a maintainer adds to swap lir::search
// (pipeline.hpp:86-87) for the B200 engine: it takes and returns the lir
// types, so call sites change from
//
//     lir::SearchResult r = lir::search(index, q, params, options);
// to
//     plaid_lir::Engine engine(index);            // once: index -> HBM
//     lir::SearchResult r = engine.search(q, params, options);
//
// and errors keep their lir::ErrorCode (a plaid_status is the ErrorCode + 1,
// error.hpp:8-26); CUDA/NCCL failures and requests outside the engine's
// envelope surface as std::runtime_error.  Timings in the returned StageTrace
// come from CUDA events (pipeline.hpp:23-43 fields, in milliseconds) when the
// Engine is created with record_times.
#pragma once

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <lir/error.hpp>
#include <lir/index.hpp>
#include <lir/pipeline.hpp>
#include <lir/types.hpp>

#include "plaid.h"

namespace plaid_lir {

inline void check(plaid_status st) {
    if (st == PLAID_OK) return;
    const std::string msg = plaid_last_error();
    if (st >= PLAID_DIMENSION_MISMATCH && st <= PLAID_IO_ERROR)
        throw lir::Error(static_cast<lir::ErrorCode>(int(st) - 1), msg);
    throw std::runtime_error(std::string(plaid_status_name(int(st))) + ": " + msg);
}

// lir::CompressedIndex (index.hpp:60-85) -> the C-ABI view (no copies).
inline plaid_index_desc describe(const lir::CompressedIndex& ix) {
    plaid_index_desc d{};
    d.dim = ix.dim;
    d.nbits = ix.nbits;
    d.num_centroids = ix.centroids.num_centroids;
    d.num_passages = ix.num_passages();
    d.num_embeddings = ix.num_embeddings();
    d.centroids = ix.centroids.data.data();
    d.codes = ix.codes.data();
    d.residuals = ix.residuals.view().data();
    d.doclens = ix.doclens.data();
    d.ivf_offsets = ix.ivf.offsets.data();
    d.ivf_postings = ix.ivf.postings.data();
    d.bucket_cutoffs = ix.quantizer.bucket_cutoffs.data();
    d.bucket_weights = ix.quantizer.bucket_weights.data();
    return d;
}

// Thread safety: lir::search is a reentrant free function over an immutable
// index (index.hpp:57-59).  An Engine owns ONE plaid_searcher (stream,
// scratch, pinned staging), so Engine::search serialises its callers on a
// mutex; for concurrent queries create one Engine per host thread (each
// uploads its own index copy) or use the C ABI directly with one
// plaid_searcher per thread over a shared plaid_index.
class Engine {
public:
    // Uploads the index to `device` (validate: re-run validate_index's
    // invariants on the way, index.cpp:12-84) and creates one searcher.
    // record_times fills StageTrace's *_ms fields from CUDA events between
    // the stages; it costs ~40 us per query (events break the programmatic
    // dependent launch chain), so it is off unless asked for.
    // use_graphs: each (rows, params) launch sequence is captured once as a
    // CUDA graph and replayed (one launch call per query instead of ~14;
    // cfg2 end to end 6.6k -> 6.8k queries/s).
    explicit Engine(const lir::CompressedIndex& index, int device = 0,
                    plaid_score_mode mode = PLAID_SCORES_TENSOR, bool validate = false,
                    bool record_times = false, bool use_graphs = true) {
        const plaid_index_desc d = describe(index);
        check(plaid_index_from_host(&d, device, validate ? 1 : 0, &index_));
        plaid_searcher_config cfg{};
        cfg.score_mode = mode;
        cfg.record_times = record_times ? 1 : 0;
        cfg.use_graphs = use_graphs ? 1 : 0;
        const plaid_status st = plaid_searcher_create(index_, device, &cfg, &searcher_);
        if (st != PLAID_OK) {
            plaid_index_close(index_);
            check(st);
        }
    }
    ~Engine() {
        plaid_searcher_destroy(searcher_);
        plaid_index_close(index_);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // lir::search (pipeline.hpp:86-87): same validation order (query, then
    // params), same result order (score desc, pid asc), same trace counters.
    // options.threads is accepted and ignored (the grid size is internal).
    lir::SearchResult search(const lir::QueryMatrix& q, const lir::SearchParams& params,
                             const lir::SearchOptions& options = {}) const {
        const plaid_params p{params.k, params.nprobe, params.t_cs, params.ndocs, options.disable_filter ? 1 : 0};
        std::vector<uint32_t> ids(params.k ? params.k : 1);
        std::vector<float> scores(ids.size());
        uint64_t n = 0;
        plaid_trace t{};
        {
            std::lock_guard<std::mutex> lock(mu_);
            check(plaid_search(searcher_, q.data.data(), q.rows, q.dim, &p, ids.data(), scores.data(), &n, &t));
        }
        return to_result(std::move(ids), std::move(scores), n, t);
    }

    // lir::SearchResult from the C ABI's outputs (pipeline.hpp:50-53).
    static lir::SearchResult to_result(std::vector<uint32_t> ids, std::vector<float> scores, uint64_t n,
                                       const plaid_trace& t) {
        lir::SearchResult r;
        ids.resize(n);
        scores.resize(n);
        r.topk.passage_ids = std::move(ids);
        r.topk.scores = std::move(scores);
        r.trace.stage1_candidates = t.stage1_candidates;
        r.trace.stage2_out = t.stage2_out;
        r.trace.stage3_out = t.stage3_out;
        r.trace.final_out = t.final_out;
        r.trace.candidate_generation_ms = t.candidate_generation_ms;
        r.trace.stage2_ms = t.stage2_ms;
        r.trace.stage3_ms = t.stage3_ms;
        r.trace.lookup_ms = t.lookup_ms;
        r.trace.decompression_ms = t.decompression_ms;
        r.trace.scoring_ms = t.scoring_ms;
        r.trace.total_ms = t.total_ms;
        r.trace.centroid_matmul_count = t.centroid_matmul_count;
        r.trace.stage2_rows_gathered = t.stage2_rows_gathered;
        r.trace.stage3_rows_gathered = t.stage3_rows_gathered;
        r.trace.decompressed_passages = t.decompressed_passages;
        return r;
    }

private:
    plaid_index* index_ = nullptr;
    plaid_searcher* searcher_ = nullptr;
    mutable std::mutex mu_;
};

// lir::search over the same index split by passage range across several GPUs
// of one node: shard g = passages [N g / G, N (g+1) / G) on
// devices[g] (devices may repeat), searched by plaid_sharded_* (on-device
// all-gathers over NVLink peer access).  global_exact = true gives exactly
// lir::search's result and trace; false = per-shard search + top-k merge.
class ShardedEngine {
public:
    ShardedEngine(const lir::CompressedIndex& index, const std::vector<int>& devices,
                  plaid_score_mode mode = PLAID_SCORES_TENSOR, bool global_exact = true) {
        if (devices.empty()) throw std::invalid_argument("ShardedEngine needs at least one device");
        const plaid_index_desc d = describe(index);
        const uint64_t N = d.num_passages, G = devices.size();
        try {
            for (uint64_t g = 0; g < G; ++g) {
                plaid_index* ix = nullptr;
                check(plaid_index_from_host_shard(&d, N * g / G, N * (g + 1) / G, devices[g], &ix));
                shards_.push_back(ix);
            }
            plaid_searcher_config cfg{};
            cfg.score_mode = mode;
            check(plaid_sharded_create(shards_.data(), uint32_t(G), &cfg,
                                       global_exact ? PLAID_SHARD_GLOBAL_EXACT : PLAID_SHARD_LOCAL, &sharded_));
        } catch (...) {
            release();
            throw;
        }
    }
    ~ShardedEngine() { release(); }
    ShardedEngine(const ShardedEngine&) = delete;
    ShardedEngine& operator=(const ShardedEngine&) = delete;

    lir::SearchResult search(const lir::QueryMatrix& q, const lir::SearchParams& params,
                             const lir::SearchOptions& options = {}) const {
        const plaid_params p{params.k, params.nprobe, params.t_cs, params.ndocs, options.disable_filter ? 1 : 0};
        std::vector<uint32_t> ids(params.k ? params.k : 1);
        std::vector<float> scores(ids.size());
        uint64_t n = 0;
        plaid_trace t{};
        {
            std::lock_guard<std::mutex> lock(mu_);
            check(plaid_sharded_search(sharded_, q.data.data(), q.rows, q.dim, &p, ids.data(), scores.data(), &n,
                                       &t));
        }
        return Engine::to_result(std::move(ids), std::move(scores), n, t);
    }

private:
    void release() {
        if (sharded_) plaid_sharded_destroy(sharded_);
        sharded_ = nullptr;
        for (plaid_index* ix : shards_) plaid_index_close(ix);
        shards_.clear();
    }
    std::vector<plaid_index*> shards_;
    plaid_sharded* sharded_ = nullptr;
    mutable std::mutex mu_;
};

}  // namespace plaid_lir
