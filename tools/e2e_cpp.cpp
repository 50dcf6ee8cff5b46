// e2e_cpp.cpp — end-to-end latency of the C++ drop-in (include/plaid_lir.hpp).
//
// A program written against the reference searcher builds a
// lir::CompressedIndex (here: the synthetic corpus of SURVEY.md §8d from the
// checker-side generator oracle/libsynth_oracle.so and the reference's own
// lir::build_inverted_list) and swaps lir::search for plaid_lir::Engine::search.
// Timed per query, host clock: Engine::search with a host lir::QueryMatrix —
// validation, H2D of Q, the 14-kernel search, D2H of the top-k and the
// lir::SearchResult construction; L2 is flushed (256 MiB write) before every
// query, outside the timed region, as in bench.py.  Prints one JSON line.
//
//   e2e_cpp <N> <K> <nbits> <mean_len> <k> <steps> <warmup> [tensor=1] [graphs=1]
//
// Built by oracle/Makefile (target e2e) because it needs the reference
// headers; the binary travels to the GPU box in oracle/_ref/.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include <cuda_runtime.h>

#include "lir/indexer.hpp"
#include "lir/pipeline.hpp"
#include "plaid_lir.hpp"

extern "C" {
void osyn_centroids(uint64_t K, uint32_t dim, uint64_t seed, float* out, int threads);
void osyn_doclens(uint64_t N, uint64_t pid_base, uint32_t min_len, uint32_t max_len, uint64_t seed, uint32_t* out,
                  int threads);
void osyn_codes(const uint32_t* doclens, const uint64_t* offsets, uint64_t N, uint64_t pid_base, uint64_t K,
                double repeat, uint64_t seed, uint32_t* codes, int threads);
void osyn_residuals(const uint64_t* offsets, uint64_t N, uint64_t pid_base, uint64_t bytes_per_token, uint64_t seed,
                    uint8_t* out, int threads);
int osyn_quantizer(uint32_t nbits, float* cutoffs, float* weights);
void osyn_queries(const float* centroids, uint32_t dim, const uint32_t* codes, const uint8_t* residuals,
                  uint32_t nbits, const float* weights, const uint32_t* doclens, const uint64_t* offsets, uint64_t N,
                  uint64_t nq, uint32_t qlen, double noise, uint64_t seed, float* out);
}

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: e2e_cpp N K nbits mean_len k steps warmup [tensor]\n");
        return 2;
    }
    const uint64_t N = std::strtoull(argv[1], nullptr, 10), K = std::strtoull(argv[2], nullptr, 10);
    const uint32_t nbits = uint32_t(std::atoi(argv[3])), mean_len = uint32_t(std::atoi(argv[4]));
    const uint64_t k = std::strtoull(argv[5], nullptr, 10);
    const int steps = std::atoi(argv[6]), warmup = std::atoi(argv[7]);
    const bool tensor = argc < 9 || std::atoi(argv[8]) != 0;
    const bool graphs = argc < 10 || std::atoi(argv[9]) != 0;
    const uint32_t dim = 128, spread = 16;

    // the synthetic corpus (same streams and seeds as bench.py / generate_index)
    lir::CompressedIndex ix;
    ix.dim = dim;
    ix.nbits = nbits;
    ix.centroids.num_centroids = K;
    ix.centroids.dim = dim;
    ix.centroids.data.resize(K * dim);
    osyn_centroids(K, dim, 11, ix.centroids.data.data(), 0);
    ix.doclens.resize(N);
    osyn_doclens(N, 0, mean_len - spread, mean_len + spread, 5, ix.doclens.data(), 0);
    std::vector<uint64_t> off(N + 1, 0);
    for (uint64_t p = 0; p < N; ++p) off[p + 1] = off[p] + ix.doclens[p];
    ix.codes.resize(off[N]);
    osyn_codes(ix.doclens.data(), off.data(), N, 0, K, 0.28, 99, ix.codes.data(), 0);
    const uint64_t bpt = uint64_t(nbits) * dim / 8;
    std::vector<uint8_t> res(off[N] * bpt);
    osyn_residuals(off.data(), N, 0, bpt, 7, res.data(), 0);
    ix.residuals = lir::ResidualStore::from_vector(std::move(res));
    ix.ivf = lir::build_inverted_list(ix.codes, ix.doclens, K);  // the reference's own builder
    float cut[16] = {}, w[16] = {};
    osyn_quantizer(nbits, cut, w);
    ix.quantizer.nbits = nbits;
    ix.quantizer.bucket_cutoffs.assign(cut, cut + (1u << nbits) - 1);
    ix.quantizer.bucket_weights.assign(w, w + (1u << nbits));
    lir::finalize_derived(ix);
    const uint64_t nq = uint64_t(steps + warmup);
    std::vector<float> qs(nq * 32 * dim);
    osyn_queries(ix.centroids.data.data(), dim, ix.codes.data(), ix.residuals.view().data(), nbits, w,
                 ix.doclens.data(), off.data(), N, nq, 32, 0.03, 1234, qs.data());

    try {
        const plaid_lir::Engine engine(ix, 0, tensor ? PLAID_SCORES_TENSOR : PLAID_SCORES_EXACT, false, false, graphs);
        const lir::SearchParams p = lir::default_params_for_k(k);
        std::vector<double> lat;
        uint64_t returned = 0;
        void* flush = nullptr;
        if (cudaMalloc(&flush, 256ull << 20) != cudaSuccess) throw std::runtime_error("flush buffer");
        for (uint64_t j = 0; j < nq; ++j) {
            lir::QueryMatrix q;
            q.rows = 32;
            q.dim = dim;
            q.data.assign(qs.begin() + j * 32 * dim, qs.begin() + (j + 1) * 32 * dim);
            cudaMemset(flush, int(j & 0xFF), 256ull << 20);
            cudaDeviceSynchronize();
            const auto t0 = std::chrono::steady_clock::now();
            const lir::SearchResult r = engine.search(q, p);
            const auto t1 = std::chrono::steady_clock::now();
            if (j >= uint64_t(warmup)) lat.push_back(std::chrono::duration<double>(t1 - t0).count());
            returned += r.topk.passage_ids.size();
        }
        cudaFree(flush);
        std::vector<double> sorted = lat;
        std::sort(sorted.begin(), sorted.end());
        const double total = std::accumulate(lat.begin(), lat.end(), 0.0);
        std::printf("{\"value\": %.3f, \"unit\": \"queries/s\", \"p50_ms\": %.4f, \"mean_ms\": %.4f, \"steps\": %d, "
                    "\"results\": %llu, \"path\": \"C++ plaid_lir::Engine::search (lir::QueryMatrix in host memory "
                    "-> lir::SearchResult), host clock per query, L2 flushed before each\", \"score_mode\": \"%s\", "
                    "\"graphs\": %s}\n",
                    lat.size() / total, 1e3 * sorted[sorted.size() / 2], 1e3 * total / lat.size(), steps,
                    (unsigned long long)returned, tensor ? "tensor" : "exact", graphs ? "true" : "false");
        return 0;
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
}
