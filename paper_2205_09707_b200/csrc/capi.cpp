// capi.cpp — the extern "C" boundary declared in include/plaid.h.
// Every entry point catches plaid::Error / std::exception and maps it to a
// plaid_status with a thread-local message (lir::Error carries the same code,
// error.hpp:51-61).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"
#include "storage.hpp"
#include "encode.hpp"

struct plaid_index {
    std::unique_ptr<plaid::DeviceIndex> impl;
};
struct plaid_searcher {
    std::unique_ptr<plaid::Searcher> impl;
};
struct plaid_batch {
    std::unique_ptr<plaid::BatchSearcher> impl;
};
struct plaid_sharded {
    std::unique_ptr<plaid::ShardedSearcher> impl;
};

namespace {

thread_local std::string g_err;

template <typename Fn>
plaid_status guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return PLAID_OK;
    } catch (const plaid::Error& e) {
        g_err = e.what();
        return static_cast<plaid_status>(e.status());
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return PLAID_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PLAID_CUDA_ERROR;
    }
}

plaid_searcher_config default_config() {
    plaid_searcher_config c{};
    c.score_mode = PLAID_SCORES_EXACT;
    c.record_times = 1;
    c.use_graphs = 0;
    return c;
}

void need(const void* p, const char* what) {
    if (!p) plaid::fail(PLAID_INVALID_PARAMS, std::string(what) + " is NULL");
}

}  // namespace

extern "C" {

const char* plaid_last_error(void) { return g_err.c_str(); }

int plaid_abi_version(void) { return PLAID_ABI_VERSION; }

// error.hpp:28-49
const char* plaid_status_name(int status) {
    switch (status) {
        case PLAID_OK: return "Ok";
        case PLAID_DIMENSION_MISMATCH: return "DimensionMismatch";
        case PLAID_NOT_NORMALIZED: return "NotNormalized";
        case PLAID_TOO_FEW_POINTS: return "TooFewPoints";
        case PLAID_PACKING_UNSUPPORTED: return "PackingUnsupported";
        case PLAID_EMPTY_CORPUS: return "EmptyCorpus";
        case PLAID_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
        case PLAID_LENGTH_NOT_PACKABLE: return "LengthNotPackable";
        case PLAID_EMPTY_PASSAGE_RANGE: return "EmptyPassageRange";
        case PLAID_INVALID_PARAMS: return "InvalidParams";
        case PLAID_CHECKSUM_MISMATCH: return "ChecksumMismatch";
        case PLAID_UNSUPPORTED_VERSION: return "UnsupportedVersion";
        case PLAID_INVARIANT_VIOLATION: return "InvariantViolation";
        case PLAID_HEADER_MISMATCH: return "HeaderMismatch";
        case PLAID_NORMALIZATION_ERROR: return "NormalizationError";
        case PLAID_LENGTH_MISMATCH: return "LengthMismatch";
        case PLAID_UNKNOWN_QUERY_ID: return "UnknownQueryId";
        case PLAID_IO_ERROR: return "IoError";
        case PLAID_CUDA_ERROR: return "CudaError";
        case PLAID_NCCL_ERROR: return "NcclError";
        case PLAID_UNSUPPORTED: return "Unsupported";
        case PLAID_OUT_OF_MEMORY: return "OutOfMemory";
    }
    return "UnknownError";
}

plaid_status plaid_validate_query(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim) {
    return guarded([&] { plaid::validate_query_host(q, rows, dim, index_dim); });
}

plaid_status plaid_validate_params(const plaid_params* p, uint64_t num_centroids) {
    return guarded([&] {
        need(p, "params");
        plaid::validate_params_host(*p, num_centroids);
    });
}

void plaid_default_params_for_k(uint64_t k, plaid_params* out) { plaid::default_params_for_k(k, out); }

uint64_t plaid_stage3_width(const plaid_params* p) { return plaid::stage3_width(*p); }

plaid_status plaid_index_from_host(const plaid_index_desc* desc, int device, int validate,
                                   plaid_index** out) {
    return guarded([&] {
        need(desc, "desc");
        need(out, "out");
        *out = nullptr;
        if (validate) plaid::validate_index_host(*desc);
        auto* h = new plaid_index();
        try {
            h->impl = std::make_unique<plaid::DeviceIndex>(*desc, device, 0);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

plaid_status plaid_index_from_host_at(const plaid_index_desc* desc, uint64_t pid_base, int device,
                                      plaid_index** out) {
    return guarded([&] {
        need(desc, "desc");
        need(out, "out");
        *out = nullptr;
        if (pid_base + desc->num_passages > 0xFFFFFFFFull)
            plaid::fail(PLAID_INVALID_PARAMS, "global passage ids must fit in 32 bits");
        auto* h = new plaid_index();
        try {
            h->impl = std::make_unique<plaid::DeviceIndex>(*desc, device, pid_base);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

// Passage-range shard: [pid_begin, pid_end) with a local IVF (postings rebased
// to local ids; each centroid's slice is a contiguous run of its sorted list).
plaid_status plaid_index_from_host_shard(const plaid_index_desc* desc, uint64_t pid_begin,
                                         uint64_t pid_end, int device, plaid_index** out) {
    return guarded([&] {
        need(desc, "desc");
        need(out, "out");
        *out = nullptr;
        if (pid_begin >= pid_end || pid_end > desc->num_passages)
            plaid::fail(PLAID_INVALID_PARAMS, "empty or out-of-range shard");
        const uint64_t K = desc->num_centroids;
        uint64_t t0 = 0;
        for (uint64_t p = 0; p < pid_begin; ++p) t0 += desc->doclens[p];
        uint64_t t1 = t0;
        for (uint64_t p = pid_begin; p < pid_end; ++p) t1 += desc->doclens[p];
        std::vector<uint64_t> offs(K + 1, 0);
        std::vector<uint32_t> post;
        for (uint64_t c = 0; c < K; ++c) {
            const uint32_t* b = desc->ivf_postings + desc->ivf_offsets[c];
            const uint32_t* e = desc->ivf_postings + desc->ivf_offsets[c + 1];
            const uint32_t* lo = std::lower_bound(b, e, uint32_t(pid_begin));
            const uint32_t* hi = std::lower_bound(lo, e, uint32_t(pid_end));
            for (const uint32_t* x = lo; x < hi; ++x) post.push_back(uint32_t(*x - pid_begin));
            offs[c + 1] = post.size();
        }
        plaid_index_desc d = *desc;
        d.num_passages = pid_end - pid_begin;
        d.num_embeddings = t1 - t0;
        d.codes = desc->codes + t0;
        d.residuals = desc->residuals + t0 * (uint64_t(desc->nbits) * desc->dim / 8);
        d.doclens = desc->doclens + pid_begin;
        d.ivf_offsets = offs.data();
        d.ivf_postings = post.data();
        auto* h = new plaid_index();
        try {
            h->impl = std::make_unique<plaid::DeviceIndex>(d, device, pid_begin);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

plaid_status plaid_index_validate(plaid_index* index) {
    return guarded([&] {
        need(index, "index");
        index->impl->validate_device();
    });
}

void plaid_index_close(plaid_index* index) { delete index; }

void plaid_index_info(const plaid_index* index, uint64_t out[8]) {
    const auto& v = index->impl->view();
    out[0] = v.dim;
    out[1] = v.nbits;
    out[2] = v.K;
    out[3] = v.N;
    out[4] = v.T;
    out[5] = v.P;
    out[6] = index->impl->pid_base();
    out[7] = index->impl->bytes();
}

plaid_status plaid_searcher_create(plaid_index* index, int device, const plaid_searcher_config* cfg,
                                   plaid_searcher** out) {
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        const plaid_searcher_config c = cfg ? *cfg : default_config();
        auto* h = new plaid_searcher();
        try {
            h->impl = std::make_unique<plaid::Searcher>(index ? index->impl.get() : nullptr, device, c);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void plaid_searcher_destroy(plaid_searcher* s) { delete s; }

plaid_status plaid_index_save(const plaid_index_desc* desc, const char* dir, uint64_t rng_seed) {
    return guarded([&] {
        need(desc, "desc");
        need(dir, "dir");
        plaid::save_index(*desc, dir, rng_seed);
    });
}

plaid_status plaid_index_open(const char* dir, int device, uint32_t flags, plaid_index** out) {
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        need(dir, "dir");
        auto* h = new plaid_index();
        try {
            h->impl.reset(plaid::open_index(dir, device, flags));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

uint64_t plaid_checksum(const void* data, uint64_t bytes) { return plaid::checksum_host(data, bytes); }

plaid_status plaid_encode(const plaid_encode_desc* in, int device, uint32_t* codes, uint8_t* residuals,
                          uint64_t* ivf_offsets, uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings) {
    return guarded([&] {
        need(in, "in");
        need(num_postings, "num_postings");
        *num_postings = 0;
        plaid::encode_host(*in, device, codes, residuals, ivf_offsets, ivf_postings, postings_cap, num_postings);
    });
}



plaid_status plaid_search(plaid_searcher* s, const float* q, uint64_t rows, uint64_t dim,
                          const plaid_params* params, uint32_t* out_pids, float* out_scores,
                          uint64_t* out_n, plaid_trace* trace) {
    return guarded([&] {
        need(s, "searcher");
        need(params, "params");
        need(out_n, "out_n");
        *out_n = 0;
        need(q, "q");
        need(out_pids, "out_pids");
        need(out_scores, "out_scores");
        s->impl->search(q, rows, dim, *params, out_pids, out_scores, out_n, trace);
    });
}

plaid_status plaid_search_batch(plaid_searcher* s, const float* q, uint64_t nq, uint64_t rows,
                                uint64_t dim, const plaid_params* params, uint32_t* out_pids,
                                float* out_scores, uint64_t* out_n, plaid_trace* traces) {
    return guarded([&] {
        need(s, "searcher");
        need(params, "params");
        for (uint64_t j = 0; j < nq; ++j)
            s->impl->search(q + j * rows * dim, rows, dim, *params, out_pids + j * params->k,
                            out_scores + j * params->k, out_n + j, traces ? traces + j : nullptr);
    });
}

plaid_status plaid_search_device(plaid_searcher* s, const float* d_q, uint64_t nq, uint64_t rows,
                                 uint64_t dim, const plaid_params* params, uint32_t* d_pids,
                                 float* d_scores, uint64_t* d_n, uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        need(params, "params");
        s->impl->search_device(d_q, nq, rows, dim, *params, d_pids, d_scores, d_n,
                               reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_batch_create(plaid_index* index, int device, const plaid_searcher_config* cfg, uint32_t lanes,
                                plaid_batch** out) {
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        need(index, "index");
        const plaid_searcher_config c = cfg ? *cfg : default_config();
        auto* h = new plaid_batch();
        try {
            h->impl = std::make_unique<plaid::BatchSearcher>(index->impl.get(), device, c, lanes);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void plaid_batch_destroy(plaid_batch* b) { delete b; }

plaid_status plaid_batch_search(plaid_batch* b, const float* q, uint64_t nq, uint64_t rows, uint64_t dim,
                                const plaid_params* params, uint32_t* out_pids, float* out_scores, uint64_t* out_n) {
    return guarded([&] {
        need(b, "batch");
        need(params, "params");
        if (nq) {
            need(q, "q");
            need(out_pids, "out_pids");
            need(out_scores, "out_scores");
            need(out_n, "out_n");
        }
        b->impl->search(q, nq, rows, dim, *params, out_pids, out_scores, out_n);
    });
}

plaid_status plaid_batch_search_device(plaid_batch* b, const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim,
                                       const plaid_params* params, uint32_t* d_pids, float* d_scores, uint64_t* d_n,
                                       uint64_t stream) {
    return guarded([&] {
        need(b, "batch");
        need(params, "params");
        b->impl->search_device(d_q, nq, rows, dim, *params, d_pids, d_scores, d_n,
                               reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_batch_sync(plaid_batch* b) {
    return guarded([&] {
        need(b, "batch");
        b->impl->sync();
    });
}

uint64_t plaid_batch_last_launches(const plaid_batch* b) { return b ? b->impl->last_launches() : 0; }

plaid_status plaid_batch_counters(plaid_batch* b, uint64_t* out, uint64_t nq) {
    return guarded([&] {
        need(b, "batch");
        need(out, "out");
        b->impl->wave_counters(out, nq);
    });
}

plaid_status plaid_batch_wave_scores(plaid_batch* b, uint64_t j, float* out) {
    return guarded([&] {
        need(b, "batch");
        need(out, "out");
        b->impl->wave_scores(j, out);
    });
}

// Debug: per-query phase timeline of the last wave batch (PLAID_WAVE_TRACE=1).
plaid_status plaid_debug_wave_trace(plaid_batch* b, uint64_t* out, uint64_t nq) {
    return guarded([&] {
        need(b, "batch");
        need(out, "out");
        b->impl->wave_trace(out, nq);
    });
}

uint32_t plaid_batch_wave_slots(const plaid_batch* b) { return b ? b->impl->wave_slots() : 0; }

int plaid_batch_last_was_wave(const plaid_batch* b) { return b && b->impl->last_was_wave() ? 1 : 0; }

plaid_status plaid_merge_topk_rows_device(plaid_searcher* s, const uint32_t* d_rows, uint64_t shards, uint64_t k,
                                          uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n,
                                          uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->merge_topk_rows_device(d_rows, shards, k, d_out_pids, d_out_scores, d_out_n,
                                        reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_shard_phase1_device(plaid_searcher* s, const float* d_q, uint64_t rows, uint64_t dim,
                                       const plaid_params* params, uint64_t* d_x2, uint64_t stride2,
                                       uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        need(params, "params");
        s->impl->shard_phase1(d_q, rows, dim, *params, d_x2, stride2, reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_shard_phase2_device(plaid_searcher* s, const uint64_t* d_g2, uint64_t shards,
                                       uint64_t* d_x3, uint64_t stride3, uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->shard_phase2(d_g2, shards, d_x3, stride3, reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_shard_phase3_device(plaid_searcher* s, const uint64_t* d_g3, uint64_t shards,
                                       uint32_t* d_pids, float* d_scores, uint64_t* d_n, uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->shard_phase3(d_g3, shards, d_pids, d_scores, d_n, reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_searcher_trace_counters_device(plaid_searcher* s, uint64_t* d_out, uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->trace_counters_device(d_out, reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_searcher_sync(plaid_searcher* s) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->sync();
    });
}

uint64_t plaid_searcher_last_launches(const plaid_searcher* s) { return s->impl->last_launches(); }

plaid_status plaid_searcher_phase_ms(plaid_searcher* s, double out[7]) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->phase_ms(out);
    });
}

plaid_status plaid_merge_topk(plaid_searcher* s, const uint32_t* pids, const float* scores,
                              const uint64_t* counts, uint64_t shards, uint64_t stride, uint64_t k,
                              uint32_t* out_pids, float* out_scores, uint64_t* out_n) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->merge_topk(pids, scores, counts, shards, stride, k, out_pids, out_scores, out_n);
    });
}

plaid_status plaid_merge_topk_device(plaid_searcher* s, const uint32_t* d_pids, const float* d_scores,
                                     const uint64_t* d_counts, uint64_t shards, uint64_t stride,
                                     uint64_t k, uint32_t* d_out_pids, float* d_out_scores,
                                     uint64_t* d_out_n, uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        s->impl->merge_topk_device(d_pids, d_scores, d_counts, shards, stride, k, d_out_pids,
                                   d_out_scores, d_out_n, reinterpret_cast<cudaStream_t>(stream));
    });
}

plaid_status plaid_compute_centroid_scores(plaid_searcher* s, const float* q, uint64_t rows,
                                           uint64_t dim, float* scores, float* row_max) {
    return guarded([&] { s->impl->compute_centroid_scores(q, rows, dim, scores, row_max); });
}

plaid_status plaid_generate_candidates(plaid_searcher* s, const float* scores, uint64_t rows,
                                       uint64_t nprobe, uint32_t* out_ids, uint64_t* out_n) {
    return guarded([&] { s->impl->generate_candidates(scores, rows, nprobe, out_ids, out_n); });
}

// pipeline.cpp:89-95 (host; one comparison per centroid).
plaid_status plaid_prune_centroids(plaid_searcher* s, const float* row_max, uint64_t num_centroids,
                                   float t_cs, uint8_t* keep) {
    (void)s;
    return guarded([&] {
        for (uint64_t c = 0; c < num_centroids; ++c) keep[c] = row_max[c] >= t_cs ? 1 : 0;
    });
}

plaid_status plaid_centroid_interaction(plaid_searcher* s, const float* scores, uint64_t rows,
                                        const uint32_t* cand, uint64_t n, const uint8_t* mask,
                                        float* out_scores, uint64_t* rows_gathered) {
    return guarded([&] { s->impl->centroid_interaction(scores, rows, cand, n, mask, out_scores, rows_gathered); });
}

plaid_status plaid_select_top(plaid_searcher* s, const uint32_t* ids, const float* scores, uint64_t n,
                              uint64_t keep, uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    return guarded([&] { s->impl->select_top(ids, scores, n, keep, out_ids, out_scores, out_n); });
}

plaid_status plaid_rank_final(plaid_searcher* s, const float* q, uint64_t rows, const uint32_t* cand,
                              uint64_t n, uint64_t k, uint32_t* out_ids, float* out_scores,
                              uint64_t* out_n) {
    return guarded([&] { s->impl->rank_final(q, rows, cand, n, k, out_ids, out_scores, out_n); });
}

plaid_status plaid_reconstruct(plaid_searcher* s, const uint32_t* codes, uint64_t n,
                               const uint8_t* residuals, float* out) {
    return guarded([&] { s->impl->reconstruct(codes, n, residuals, out); });
}

// residual_codec.cpp:42-59
plaid_status plaid_lut_build(uint32_t nbits, uint8_t* table) {
    return guarded([&] {
        if (nbits != 1 && nbits != 2 && nbits != 4) plaid::fail(PLAID_PACKING_UNSUPPORTED, "nbits not in {1,2,4}");
        const uint32_t per = 8 / nbits, mask = (1u << nbits) - 1;
        for (uint32_t v = 0; v < 256; ++v)
            for (uint32_t j = 0; j < per; ++j) table[v * per + j] = uint8_t((v >> (nbits * j)) & mask);
    });
}

plaid_status plaid_unpack_via_lut(plaid_searcher* s, const uint8_t* packed, uint64_t n, uint32_t nbits,
                                  uint8_t* out) {
    return guarded([&] { s->impl->unpack(packed, n, nbits, out); });
}

// residual_codec.cpp:61-84 (index-build side)
plaid_status plaid_pack_residual(const uint8_t* idx, uint64_t n, uint32_t nbits, uint8_t* out) {
    return guarded([&] {
        if (nbits != 1 && nbits != 2 && nbits != 4) plaid::fail(PLAID_PACKING_UNSUPPORTED, "nbits not in {1,2,4}");
        const uint32_t per = 8 / nbits;
        if (n % per != 0) plaid::fail(PLAID_LENGTH_NOT_PACKABLE, "indices not divisible by 8/nbits");
        std::memset(out, 0, n / per);
        for (uint64_t i = 0; i < n; ++i) {
            if (idx[i] >= (1u << nbits)) plaid::fail(PLAID_INDEX_OUT_OF_RANGE, "bucket index out of range");
            out[i / per] |= uint8_t(idx[i] << (nbits * (i % per)));
        }
    });
}

plaid_status plaid_maxsim_packed(plaid_searcher* s, const float* scores, uint64_t nq,
                                 const uint64_t* offsets, uint64_t np, float* out) {
    return guarded([&] { s->impl->maxsim_packed(scores, nq, offsets, np, out); });
}

plaid_status plaid_maxsim_embeddings(plaid_searcher* s, const float* q, uint64_t rows, uint64_t dim,
                                     const float* emb, const uint64_t* offsets, uint64_t np,
                                     float* out) {
    return guarded([&] { s->impl->maxsim_embeddings(q, rows, dim, emb, offsets, np, out); });
}

plaid_status plaid_merge_topk_batch_device(plaid_searcher* s, const uint32_t* d_pids, const float* d_scores,
                                           const uint64_t* d_counts, uint64_t shards, uint64_t batch, uint64_t k,
                                           uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n,
                                           uint64_t stream) {
    return guarded([&] {
        need(s, "searcher");
        if (k < 1) plaid::fail(PLAID_INVALID_PARAMS, "k must be >= 1");
        if (shards * k > 25600) plaid::fail(PLAID_UNSUPPORTED, "shards x k above 25600");
        plaid::DeviceGuard g(s->impl->device());
        cudaStream_t st = stream ? reinterpret_cast<cudaStream_t>(stream) : s->impl->stream();
        plaid::launch::merge_batch(d_pids, d_scores, d_counts, uint32_t(shards), uint32_t(batch), uint32_t(k),
                                   d_out_pids, d_out_scores, d_out_n, st);
        PLAID_CUDA(cudaGetLastError());
    });
}

plaid_status plaid_sharded_create(plaid_index* const* shards, uint32_t num_shards, const plaid_searcher_config* cfg,
                                  int32_t mode, plaid_sharded** out) {
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        need(shards, "shards");
        std::vector<plaid::DeviceIndex*> v;
        for (uint32_t g = 0; g < num_shards; ++g) {
            need(shards[g], "shard index");
            v.push_back(shards[g]->impl.get());
        }
        const plaid_searcher_config c = cfg ? *cfg : default_config();
        auto* h = new plaid_sharded();
        try {
            h->impl = std::make_unique<plaid::ShardedSearcher>(v, c, mode);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void plaid_sharded_destroy(plaid_sharded* s) { delete s; }

plaid_status plaid_sharded_search(plaid_sharded* s, const float* q, uint64_t rows, uint64_t dim,
                                  const plaid_params* params, uint32_t* out_pids, float* out_scores, uint64_t* out_n,
                                  plaid_trace* trace) {
    return guarded([&] {
        need(s, "sharded searcher");
        need(params, "params");
        need(out_n, "out_n");
        *out_n = 0;
        need(q, "q");
        need(out_pids, "out_pids");
        need(out_scores, "out_scores");
        s->impl->search(q, rows, dim, *params, out_pids, out_scores, out_n, trace);
    });
}

uint64_t plaid_sharded_last_launches(const plaid_sharded* s) { return s ? s->impl->last_launches() : 0; }

plaid_status plaid_index_synth(const plaid_synth_desc* desc, int device, plaid_index** out) {
    return guarded([&] {
        need(desc, "desc");
        need(out, "out");
        *out = nullptr;
        plaid::SynthSpec sp;
        sp.num_passages = desc->num_passages;
        sp.num_centroids = desc->num_centroids;
        sp.pid_base = desc->pid_base;
        sp.seed = desc->seed;
        sp.dim = desc->dim;
        sp.nbits = desc->nbits;
        sp.mean_len = desc->mean_len;
        sp.spread = desc->spread;
        sp.repeat = desc->repeat;
        auto* h = new plaid_index();
        try {
            h->impl = std::make_unique<plaid::DeviceIndex>(sp, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

plaid_status plaid_index_synth_queries(plaid_index* index, uint64_t nq, uint32_t qlen, double noise, uint64_t seed,
                                       float* out) {
    return guarded([&] {
        need(index, "index");
        need(out, "out");
        index->impl->synth_queries(nq, qlen, noise, seed, out);
    });
}

plaid_status plaid_index_export(plaid_index* index, float* centroids, uint32_t* codes, uint8_t* residuals,
                                uint32_t* doclens, uint64_t* ivf_offsets, uint32_t* ivf_postings, float* cutoffs,
                                float* weights) {
    return guarded([&] {
        need(index, "index");
        index->impl->export_host(centroids, codes, residuals, doclens, ivf_offsets, ivf_postings, cutoffs, weights);
    });
}

plaid_status plaid_build_index(const plaid_build_desc* in, int device, float* centroids, uint64_t centroids_cap,
                               uint64_t* num_centroids, float* bucket_cutoffs, float* bucket_weights, uint32_t* codes,
                               uint8_t* residuals, uint64_t* ivf_offsets, uint32_t* ivf_postings, uint64_t postings_cap,
                               uint64_t* num_postings) {
    return guarded([&] {
        need(in, "desc");
        need(in->embeddings, "embeddings");
        need(in->doclens, "doclens");
        need(num_centroids, "num_centroids");
        uint64_t T = 0;
        for (uint64_t p = 0; p < in->num_passages; ++p) T += in->doclens[p];
        if (T != in->num_embeddings) plaid::fail(PLAID_LENGTH_MISMATCH, "doclens total does not match the embedding rows");
        uint64_t k = in->num_centroids;
        if (!k && T) k = std::min<uint64_t>(uint64_t(1) << uint64_t(std::ceil(std::log2(double(T)) / 2.0)), T);
        if (k > centroids_cap) plaid::fail(PLAID_INVALID_PARAMS, "centroids capacity below K = " + std::to_string(k));
        plaid::build_index_host(in->embeddings, in->doclens, in->num_passages, in->dim, in->nbits, in->num_centroids,
                                in->kmeans_iters, in->rng_seed, device, centroids, bucket_cutoffs, bucket_weights,
                                num_centroids, codes, residuals, ivf_offsets, ivf_postings, postings_cap, num_postings);
    });
}

}  // extern "C"
