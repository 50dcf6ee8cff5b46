// lir_dropin.cpp — TEST INFRASTRUCTURE: the drop-in demonstration.
//
// Code written against the reference searcher (`lir`, compiled from
// /root/reference/proj/src into oracle/_ref/liblir_ref.so) swaps lir::search
// for plaid_lir::Engine::search (include/plaid_lir.hpp over libplaid.so) with
// no other change.  The program builds an index with the reference's own
// offline builder (lir::build_index), runs both searchers on the same queries
// and prints one line per query:  "<q> <k> <ids_equal> <score_bits_equal>
// <trace_equal> sharded <bit-exact> tensor <within tolerance>", then "OK"
// when everything matched: plaid_lir::Engine in EXACT mode and
// plaid_lir::ShardedEngine (three passage shards, global-exact) bit for bit,
// the TENSOR default within north_star's tolerance —
// tests/test_gpu_parity.py runs it on the GPU box.  Without a GPU the Engine
// constructor throws (no CPU fallback) and the program prints "NOGPU".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "lir/indexer.hpp"
#include "lir/pipeline.hpp"
#include "plaid_lir.hpp"

int main() {
    const std::size_t dim = 128, N = 400;
    std::mt19937_64 rng(7);
    std::normal_distribution<float> g(0.f, 1.f);
    std::uniform_int_distribution<uint32_t> len(8, 40);
    std::vector<uint32_t> doclens(N);
    std::size_t T = 0;
    for (auto& l : doclens) T += (l = len(rng));
    std::vector<float> topics(16 * dim);
    for (auto& x : topics) x = g(rng);
    std::vector<float> data(T * dim);
    for (std::size_t t = 0; t < T; ++t) {
        const float* tp = &topics[(rng() % 16) * dim];
        double n2 = 0;
        for (std::size_t d = 0; d < dim; ++d) {
            data[t * dim + d] = tp[d] + 0.7f * g(rng);
            n2 += double(data[t * dim + d]) * data[t * dim + d];
        }
        for (std::size_t d = 0; d < dim; ++d) data[t * dim + d] = float(data[t * dim + d] / std::sqrt(n2));
    }
    auto corpus = lir::CorpusEmbeddings::create(dim, doclens, data);
    lir::IndexConfig cfg;
    cfg.nbits = 2;
    cfg.num_centroids = 64;
    cfg.kmeans_iters = 4;
    const lir::CompressedIndex index = lir::build_index(corpus, cfg, 1);

    try {
        const plaid_lir::Engine engine(index, 0, PLAID_SCORES_EXACT, /*validate=*/true);
        // the production default (tcgen05 S_cq + stage 4) and the multi-GPU
        // drop-in (three passage shards; all on GPU 0 here)
        const plaid_lir::Engine tensor(index, 0, PLAID_SCORES_TENSOR);
        const plaid_lir::ShardedEngine sharded(index, {0, 0, 0}, PLAID_SCORES_EXACT, /*global_exact=*/true);
        bool all = true;
        for (int qi = 0; qi < 4; ++qi) {
            lir::QueryMatrix q;
            q.rows = 32;
            q.dim = dim;
            q.data.resize(32 * dim);
            for (std::size_t i = 0; i < 32; ++i) {
                const std::size_t t = rng() % T;
                double n2 = 0;
                for (std::size_t d = 0; d < dim; ++d) {
                    q.data[i * dim + d] = data[t * dim + d] + 0.05f * g(rng);
                    n2 += double(q.data[i * dim + d]) * q.data[i * dim + d];
                }
                for (std::size_t d = 0; d < dim; ++d) q.data[i * dim + d] = float(q.data[i * dim + d] / std::sqrt(n2));
            }
            for (std::size_t k : {10, 100}) {
                const lir::SearchParams p = lir::default_params_for_k(k);
                const lir::SearchResult a = lir::search(index, q, p);
                const lir::SearchResult b = engine.search(q, p);
                const bool ids = a.topk.passage_ids == b.topk.passage_ids;
                bool sc = ids && a.topk.scores && b.topk.scores && a.topk.scores->size() == b.topk.scores->size();
                for (std::size_t j = 0; sc && j < a.topk.scores->size(); ++j)
                    sc = std::memcmp(&(*a.topk.scores)[j], &(*b.topk.scores)[j], 4) == 0;
                const auto& x = a.trace;
                const auto& y = b.trace;
                const bool tr = x.stage1_candidates == y.stage1_candidates && x.stage2_out == y.stage2_out &&
                                x.stage3_out == y.stage3_out && x.final_out == y.final_out &&
                                x.centroid_matmul_count == y.centroid_matmul_count &&
                                x.stage2_rows_gathered == y.stage2_rows_gathered &&
                                x.stage3_rows_gathered == y.stage3_rows_gathered &&
                                x.decompressed_passages == y.decompressed_passages;
                // sharded: the same bits and counters as lir::search
                const lir::SearchResult c = sharded.search(q, p);
                bool sh = c.topk.passage_ids == a.topk.passage_ids && c.topk.scores && a.topk.scores &&
                          c.topk.scores->size() == a.topk.scores->size();
                for (std::size_t j = 0; sh && j < a.topk.scores->size(); ++j)
                    sh = std::memcmp(&(*a.topk.scores)[j], &(*c.topk.scores)[j], 4) == 0;
                sh = sh && c.trace.stage1_candidates == x.stage1_candidates && c.trace.stage2_out == x.stage2_out &&
                     c.trace.stage3_out == x.stage3_out && c.trace.stage2_rows_gathered == x.stage2_rows_gathered &&
                     c.trace.stage3_rows_gathered == x.stage3_rows_gathered;
                // tensor: every returned score within 1e-4 relative of the
                // reference's score of the same pid, the top-k equal up to
                // near-ties (at most 2 swapped at the boundary)
                const lir::SearchResult t = tensor.search(q, p);
                std::size_t common = 0;
                bool tol = t.topk.scores && a.topk.scores;
                for (std::size_t j = 0; tol && j < t.topk.passage_ids.size(); ++j)
                    for (std::size_t m = 0; m < a.topk.passage_ids.size(); ++m)
                        if (a.topk.passage_ids[m] == t.topk.passage_ids[j]) {
                            ++common;
                            const float ra = (*a.topk.scores)[m], rt = (*t.topk.scores)[j];
                            tol = tol && std::fabs(rt - ra) <= 1e-4f * std::fabs(ra);
                        }
                const bool ten = tol && common + 2 >= a.topk.passage_ids.size() &&
                                 t.topk.passage_ids.size() == a.topk.passage_ids.size();
                std::printf("%d %zu %d %d %d sharded %d tensor %d\n", qi, k, int(ids), int(sc), int(tr), int(sh),
                            int(ten));
                all = all && ids && sc && tr && sh && ten;
            }
        }
        // errors keep their lir::ErrorCode across the boundary
        lir::QueryMatrix bad;
        bad.rows = 1;
        bad.dim = dim;
        bad.data.assign(dim, 0.5f);
        try {
            engine.search(bad, lir::default_params_for_k(10));
            all = false;
        } catch (const lir::Error& e) {
            all = all && e.code() == lir::ErrorCode::NotNormalized;
        }
        std::printf(all ? "OK\n" : "MISMATCH\n");
        return all ? 0 : 1;
    } catch (const lir::Error& e) {
        std::printf("LIR_ERROR %s\n", e.what());
        return 3;
    } catch (const std::runtime_error& e) {
        std::printf("NOGPU %s\n", e.what());
        return 2;
    }
}
