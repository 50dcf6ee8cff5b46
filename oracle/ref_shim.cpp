// ref_shim.cpp — extern "C" face of the UNMODIFIED reference library (lir),
// compiled together with /root/reference/proj/src/*.cpp by oracle/Makefile
// into oracle/_ref/liblir_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin oracle/plaid_oracle.c and to
// produce golden vectors, and by bench.py's cpu_baseline / --impl reference
// legs to time the reference's own CPU searcher.  No reference source is
// copied; this file only converts plain arrays to lir types and calls the
// reference's public API (pipeline.hpp:55-90, residual_codec.hpp, maxsim.hpp,
// indexer.hpp, index.hpp).
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lir/index.hpp"
#include "lir/indexer.hpp"
#include "lir/maxsim.hpp"
#include "lir/pipeline.hpp"
#include "lir/residual_codec.hpp"
#include "lir/types.hpp"

#include "plaid_oracle.h"  // orc_index / orc_params / orc_trace layouts

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const lir::Error& e) {
        g_err = e.what();
        return static_cast<int>(e.code()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 102;
    }
}

lir::QueryMatrix make_query(const float* q, uint64_t rows, uint64_t dim) {
    lir::QueryMatrix m;
    m.rows = rows;
    m.dim = dim;
    m.data.assign(q, q + rows * dim);
    return m;
}

lir::SearchParams make_params(const orc_params* p) {
    lir::SearchParams s;
    s.k = p->k;
    s.nprobe = p->nprobe;
    s.t_cs = p->t_cs;
    s.ndocs = p->ndocs;
    return s;
}

lir::QuantizerSpec make_quant(uint32_t nbits, const float* cutoffs, const float* weights) {
    lir::QuantizerSpec q;
    q.nbits = nbits;
    std::size_t nb = std::size_t(1) << nbits;
    q.bucket_cutoffs.assign(cutoffs, cutoffs + nb - 1);
    q.bucket_weights.assign(weights, weights + nb);
    return q;
}

void fill_trace(const lir::StageTrace& t, orc_trace* out, double* times) {
    if (out) {
        out->stage1_candidates = t.stage1_candidates;
        out->stage2_out = t.stage2_out;
        out->stage3_out = t.stage3_out;
        out->final_out = t.final_out;
        out->centroid_matmul_count = t.centroid_matmul_count;
        out->stage2_rows_gathered = t.stage2_rows_gathered;
        out->stage3_rows_gathered = t.stage3_rows_gathered;
        out->decompressed_passages = t.decompressed_passages;
    }
    if (times) {
        times[0] = t.candidate_generation_ms;
        times[1] = t.stage2_ms;
        times[2] = t.stage3_ms;
        times[3] = t.lookup_ms;
        times[4] = t.decompression_ms;
        times[5] = t.scoring_ms;
        times[6] = t.total_ms;
    }
}

void copy_out(const lir::CandidateSet& c, uint32_t* ids, float* scores, uint64_t* n) {
    *n = c.size();
    if (c.size()) std::memcpy(ids, c.passage_ids.data(), c.size() * sizeof(uint32_t));
    if (scores && c.scores && c.size()) std::memcpy(scores, c.scores->data(), c.size() * sizeof(float));
}

// Parallel memcpy for the multi-GB arrays of the bench-scale index.
void pcopy(void* dst, const void* src, std::size_t bytes) {
    unsigned t = std::max(1u, std::thread::hardware_concurrency());
    if (bytes < (std::size_t(64) << 20)) t = 1;
    std::size_t chunk = (bytes + t - 1) / t;
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < t; ++w) {
        std::size_t b = w * chunk, e = std::min(bytes, b + chunk);
        if (b >= e) break;
        pool.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
        });
    }
    for (auto& th : pool) th.join();
}

template <typename T>
std::vector<T> vec_from(const T* p, std::size_t n) {
    std::vector<T> v(n);
    if (n) pcopy(v.data(), p, n * sizeof(T));
    return v;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Builds a lir::CompressedIndex (index.hpp:60-85) from plain arrays, then
// finalize_derived (index.cpp:7-10).  Arrays are copied.
void* ref_index_build(const orc_index* d, int* status) {
    lir::CompressedIndex* idx = nullptr;
    *status = guarded([&] {
        auto* x = new lir::CompressedIndex();
        x->dim = d->dim;
        x->nbits = d->nbits;
        x->centroids.num_centroids = d->num_centroids;
        x->centroids.dim = d->dim;
        x->centroids.data = vec_from(d->centroids, d->num_centroids * d->dim);
        x->codes = vec_from(d->codes, d->num_embeddings);
        std::size_t rb = d->num_embeddings * (std::size_t(d->nbits) * d->dim / 8);
        x->residuals = lir::ResidualStore::from_vector(vec_from(d->residuals, rb));
        x->doclens = vec_from(d->doclens, d->num_passages);
        x->ivf.offsets = vec_from(d->ivf_offsets, d->num_centroids + 1);
        x->ivf.postings = vec_from(d->ivf_postings, d->ivf_offsets[d->num_centroids]);
        x->quantizer = make_quant(d->nbits, d->bucket_cutoffs, d->bucket_weights);
        lir::finalize_derived(*x);
        idx = x;
    });
    return idx;
}

void ref_index_free(void* h) { delete static_cast<lir::CompressedIndex*>(h); }

int ref_index_validate(void* h) {
    return guarded([&] { lir::validate_index(*static_cast<lir::CompressedIndex*>(h)); });
}

int ref_search(void* h, const float* q, uint64_t rows, uint64_t dim, const orc_params* p,
               int threads, uint32_t* out_ids, float* out_scores, uint64_t* out_n,
               orc_trace* trace, double* times) {
    *out_n = 0;
    return guarded([&] {
        lir::SearchOptions opt;
        opt.threads = threads;
        opt.disable_filter = p->disable_filter != 0;
        auto r = lir::search(*static_cast<lir::CompressedIndex*>(h), make_query(q, rows, dim),
                             make_params(p), opt);
        copy_out(r.topk, out_ids, out_scores, out_n);
        fill_trace(r.trace, trace, times);
    });
}

// Runs nq queries back to back.  mode 0 = latency mode (one search at a time
// with SearchOptions.threads = threads); mode 1 = throughput mode (`threads`
// workers, each calling search with threads = 1).  Results
// land in out_ids/out_scores at stride k; per-query latencies in lat_ms.
int ref_search_many(void* h, const float* q, uint64_t nq, uint64_t rows, uint64_t dim,
                    const orc_params* p, int mode, int threads, uint32_t* out_ids,
                    float* out_scores, uint64_t* out_n, double* lat_ms) {
    auto& idx = *static_cast<lir::CompressedIndex*>(h);
    lir::SearchParams params = make_params(p);
    std::atomic<int> status{0};
    auto run_one = [&](uint64_t j, int thr) {
        auto t0 = std::chrono::steady_clock::now();
        int rc = guarded([&] {
            lir::SearchOptions opt;
            opt.threads = thr;
            opt.disable_filter = p->disable_filter != 0;
            auto r = lir::search(idx, make_query(q + j * rows * dim, rows, dim), params, opt);
            copy_out(r.topk, out_ids + j * p->k, out_scores + j * p->k, out_n + j);
        });
        if (rc) status.store(rc);
        lat_ms[j] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    if (mode == 0) {
        for (uint64_t j = 0; j < nq; ++j) run_one(j, threads);
    } else {
        std::atomic<uint64_t> next{0};
        std::vector<std::thread> pool;
        for (int w = 0; w < std::max(1, threads); ++w)
            pool.emplace_back([&] {
                for (uint64_t j; (j = next.fetch_add(1)) < nq;) run_one(j, 1);
            });
        for (auto& th : pool) th.join();
    }
    return status.load();
}

int ref_validate_query(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim) {
    return guarded([&] { lir::validate_query(make_query(q, rows, dim), index_dim); });
}

int ref_validate_params(const orc_params* p, uint64_t num_centroids) {
    return guarded([&] { lir::validate_params(make_params(p), num_centroids); });
}

void ref_default_params_for_k(uint64_t k, orc_params* out) {
    auto s = lir::default_params_for_k(k);
    out->k = s.k;
    out->nprobe = s.nprobe;
    out->t_cs = s.t_cs;
    out->ndocs = s.ndocs;
    out->disable_filter = 0;
}

uint64_t ref_stage3_width(const orc_params* p) { return lir::stage3_width(make_params(p)); }

int ref_lut_build(uint32_t nbits, uint8_t* table) {
    return guarded([&] {
        auto lut = lir::DecompressionLUT::build(nbits);
        std::memcpy(table, lut.table.data(), lut.table.size());
    });
}

int ref_pack_residual(const uint8_t* idx, uint64_t n, uint32_t nbits, uint8_t* out) {
    return guarded([&] {
        auto v = lir::pack_residual(std::span<const uint8_t>(idx, n), nbits);
        std::memcpy(out, v.data(), v.size());
    });
}

int ref_unpack_via_lut(const uint8_t* packed, uint64_t n, uint32_t nbits, uint8_t* out) {
    return guarded([&] {
        auto lut = lir::DecompressionLUT::build(nbits);
        auto v = lir::unpack_via_lut(std::span<const uint8_t>(packed, n), lut);
        std::memcpy(out, v.data(), v.size());
    });
}

int ref_reconstruct(const uint32_t* codes, uint64_t n, const uint8_t* residuals,
                    const float* centroids, uint64_t num_centroids, uint32_t dim, uint32_t nbits,
                    const float* cutoffs, const float* weights, float* out) {
    return guarded([&] {
        lir::CentroidSet cs;
        cs.num_centroids = num_centroids;
        cs.dim = dim;
        cs.data.assign(centroids, centroids + num_centroids * dim);
        auto quant = make_quant(nbits, cutoffs, weights);
        auto lut = lir::DecompressionLUT::build(nbits);
        lir::reconstruct(std::span<const uint32_t>(codes, n),
                         std::span<const uint8_t>(residuals, n * (std::size_t(nbits) * dim / 8)), cs,
                         quant, lut, std::span<float>(out, n * dim), 1);
    });
}

int ref_compute_centroid_scores(const float* q, uint64_t rows, uint64_t dim, const float* centroids,
                                uint64_t num_centroids, float* scores, float* row_max) {
    return guarded([&] {
        lir::CentroidSet cs;
        cs.num_centroids = num_centroids;
        cs.dim = dim;
        cs.data.assign(centroids, centroids + num_centroids * dim);
        auto t = lir::compute_centroid_scores(make_query(q, rows, dim), cs, 1);
        std::memcpy(scores, t.scores.data(), t.scores.size() * sizeof(float));
        std::memcpy(row_max, t.per_centroid_max.data(), t.per_centroid_max.size() * sizeof(float));
    });
}

static lir::CentroidScoreTable make_table(const float* scores, uint64_t num_centroids, uint64_t rows) {
    lir::CentroidScoreTable t;
    t.num_centroids = num_centroids;
    t.num_query_tokens = rows;
    t.scores.assign(scores, scores + num_centroids * rows);
    t.per_centroid_max.assign(num_centroids, 0.0f);
    return t;
}

int ref_generate_candidates(const float* scores, uint64_t num_centroids, uint64_t rows,
                            const uint64_t* ivf_offsets, const uint32_t* ivf_postings,
                            uint64_t nprobe, uint64_t num_passages, uint32_t* out_ids,
                            uint64_t* out_n) {
    *out_n = 0;
    return guarded([&] {
        lir::InvertedList ivf;
        ivf.offsets.assign(ivf_offsets, ivf_offsets + num_centroids + 1);
        ivf.postings.assign(ivf_postings, ivf_postings + ivf_offsets[num_centroids]);
        auto c = lir::generate_candidates(make_table(scores, num_centroids, rows), ivf, nprobe,
                                          num_passages);
        copy_out(c, out_ids, nullptr, out_n);
    });
}

void ref_prune_centroids(const float* row_max, uint64_t num_centroids, float t_cs, uint8_t* keep) {
    lir::CentroidScoreTable t;
    t.num_centroids = num_centroids;
    t.num_query_tokens = 1;
    t.per_centroid_max.assign(row_max, row_max + num_centroids);
    auto k = lir::prune_centroids(t, t_cs);
    std::memcpy(keep, k.data(), k.size());
}

int ref_centroid_interaction(void* h, const float* scores, uint64_t rows, const uint32_t* cand,
                             uint64_t n, const uint8_t* mask, float* out_scores,
                             uint64_t* rows_gathered) {
    return guarded([&] {
        auto& idx = *static_cast<lir::CompressedIndex*>(h);
        lir::CandidateSet c;
        c.passage_ids.assign(cand, cand + n);
        std::vector<uint8_t> m;
        if (mask) m.assign(mask, mask + idx.centroids.num_centroids);
        uint64_t g = 0;
        auto out = lir::centroid_interaction(c, idx, make_table(scores, idx.centroids.num_centroids, rows),
                                             mask ? &m : nullptr, 1, &g);
        std::memcpy(out_scores, out.scores->data(), n * sizeof(float));
        if (rows_gathered) *rows_gathered = g;
    });
}

int ref_select_top(const uint32_t* ids, const float* scores, uint64_t n, uint64_t keep,
                   uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    *out_n = 0;
    return guarded([&] {
        lir::CandidateSet c;
        c.passage_ids.assign(ids, ids + n);
        c.scores.emplace(scores, scores + n);
        copy_out(lir::select_top(c, keep), out_ids, out_scores, out_n);
    });
}

int ref_maxsim_packed(const float* scores, uint64_t nq, const uint64_t* offsets, uint64_t np,
                      float* out) {
    return guarded([&] {
        lir::PackedScores ps;
        ps.num_query_tokens = nq;
        ps.offsets.assign(offsets, offsets + np + 1);
        ps.data.assign(scores, scores + offsets[np] * nq);
        auto v = lir::maxsim_packed(ps, 1);
        std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

int ref_maxsim_embeddings(const float* q, uint64_t rows, uint64_t dim, const float* emb,
                          const uint64_t* offsets, uint64_t np, float* out) {
    return guarded([&] {
        auto v = lir::maxsim_embeddings(make_query(q, rows, dim),
                                        std::span<const float>(emb, offsets[np] * dim),
                                        std::span<const uint64_t>(offsets, np + 1), 1);
        std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

int ref_rank_final(void* h, const float* q, uint64_t rows, const uint32_t* cand, uint64_t n,
                   uint64_t k, uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    *out_n = 0;
    return guarded([&] {
        auto& idx = *static_cast<lir::CompressedIndex*>(h);
        lir::CandidateSet c;
        c.passage_ids.assign(cand, cand + n);
        copy_out(lir::rank_final(c, idx, make_query(q, rows, idx.dim), k, 1), out_ids, out_scores,
                 out_n);
    });
}

// indexer.cpp:149-195 — used to check the synthetic generator's IVF.
int ref_build_inverted_list(const uint32_t* codes, uint64_t T, const uint32_t* doclens, uint64_t N,
                            uint64_t K, uint64_t* out_offsets, uint32_t* out_postings,
                            uint64_t cap, uint64_t* out_P) {
    return guarded([&] {
        auto ivf = lir::build_inverted_list(std::span<const uint32_t>(codes, T),
                                            std::span<const uint32_t>(doclens, N), K);
        *out_P = ivf.postings.size();
        std::memcpy(out_offsets, ivf.offsets.data(), (K + 1) * sizeof(uint64_t));
        if (ivf.postings.size() <= cap)
            std::memcpy(out_postings, ivf.postings.data(), ivf.postings.size() * sizeof(uint32_t));
    });
}

// indexer.cpp:197-282 — the reference's own offline build (k-means etc.), used
// only to make golden fixtures.  Returns an index handle; export with
// ref_index_export_*.
void* ref_build_index(const float* data, const uint32_t* doclens, uint64_t N, uint64_t dim,
                      uint32_t nbits, uint64_t K, uint64_t iters, uint64_t seed, int threads,
                      int* status) {
    lir::CompressedIndex* out = nullptr;
    *status = guarded([&] {
        std::vector<uint32_t> dl(doclens, doclens + N);
        uint64_t T = 0;
        for (auto l : dl) T += l;
        auto corpus = lir::CorpusEmbeddings::create(dim, dl, std::vector<float>(data, data + T * dim));
        lir::IndexConfig cfg;
        cfg.nbits = nbits;
        cfg.num_centroids = K;
        cfg.kmeans_iters = iters;
        cfg.rng_seed = seed;
        out = new lir::CompressedIndex(lir::build_index(corpus, cfg, threads));
    });
    return out;
}

void ref_index_sizes(void* h, uint64_t* sizes /* dim, nbits, K, N, T, P */) {
    auto& x = *static_cast<lir::CompressedIndex*>(h);
    sizes[0] = x.dim;
    sizes[1] = x.nbits;
    sizes[2] = x.centroids.num_centroids;
    sizes[3] = x.num_passages();
    sizes[4] = x.num_embeddings();
    sizes[5] = x.ivf.postings.size();
}

void ref_index_export(void* h, float* centroids, uint32_t* codes, uint8_t* residuals,
                      uint32_t* doclens, uint64_t* ivf_offsets, uint32_t* ivf_postings,
                      float* cutoffs, float* weights) {
    auto& x = *static_cast<lir::CompressedIndex*>(h);
    std::memcpy(centroids, x.centroids.data.data(), x.centroids.data.size() * sizeof(float));
    std::memcpy(codes, x.codes.data(), x.codes.size() * sizeof(uint32_t));
    std::memcpy(residuals, x.residuals.view().data(), x.residuals.size());
    std::memcpy(doclens, x.doclens.data(), x.doclens.size() * sizeof(uint32_t));
    std::memcpy(ivf_offsets, x.ivf.offsets.data(), x.ivf.offsets.size() * sizeof(uint64_t));
    std::memcpy(ivf_postings, x.ivf.postings.data(), x.ivf.postings.size() * sizeof(uint32_t));
    std::memcpy(cutoffs, x.quantizer.bucket_cutoffs.data(), x.quantizer.bucket_cutoffs.size() * sizeof(float));
    std::memcpy(weights, x.quantizer.bucket_weights.data(), x.quantizer.bucket_weights.size() * sizeof(float));
}

}  // extern "C"
