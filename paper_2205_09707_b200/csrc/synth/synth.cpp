// synth.cpp — deterministic synthetic PLAID index + query generator (host C++).
//
// Produces the arrays of a lir::CompressedIndex (reference index.hpp:60-85)
// directly, without k-means, following SURVEY.md §8d / Appendix A.1:
//   * centroids  K rows of normalize(N(0, I_d))                 stream (seed, c)
//   * doclens    uniform in [min_len, max_len]                   stream (seed, p)
//   * codes      per passage: with prob `repeat` reuse an earlier code of the
//                same passage, else uniform over [0, K)           stream (seed, p)
//   * residuals  uniform random bytes                            stream (seed, t)
//   * IVF        build_inverted_list semantics (indexer.cpp:149-195): per
//                centroid the sorted unique passage ids owning a token of it
//   * queries    each token = normalize(reconstruct(random token) + N(0, s^2))
// Every stream is a counter-keyed SplitMix64 (the algorithm of rng.hpp:11-56),
// so the bytes are identical for any thread count and on every host.  The
// same bytes feed the CUDA engine and the CPU reference, which is what makes
// bit-exact parity checks possible.
//
// Fixture infrastructure: used by tests/, bench.py and smoke(); it is not on
// the search path.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Rng {  // SplitMix64 stream
    uint64_t s;
    double spare = 0;
    bool have = false;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return (double(next() >> 11) + 0.5) * 0x1.0p-53; }
    uint64_t below(uint64_t bound) { return bound ? next() % bound : 0; }
    double gauss() {  // Box-Muller, one spare cached
        if (have) {
            have = false;
            return spare;
        }
        double u1 = unit(), u2 = unit();
        double r = std::sqrt(-2.0 * std::log(u1));
        double th = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(th);
        have = true;
        return r * std::cos(th);
    }
};

uint64_t stream_seed(uint64_t a, uint64_t b) {
    Rng r(a ^ (0x9E3779B97F4A7C15ULL + (b << 6) + (b >> 2)));
    return r.next();
}

unsigned nthreads(int threads) {
    if (threads > 0) return unsigned(threads);
    unsigned hc = std::thread::hardware_concurrency();
    return hc ? hc : 1;
}

template <typename Fn>
void parallel_range(uint64_t n, int threads, Fn&& fn) {
    unsigned t = std::min<uint64_t>(nthreads(threads), std::max<uint64_t>(n, 1));
    if (t <= 1) {
        fn(0, n, 0u);
        return;
    }
    uint64_t chunk = (n + t - 1) / t;
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < t; ++w) {
        uint64_t b = w * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e, w] { fn(b, e, w); });
    }
    for (auto& th : pool) th.join();
}

void normalize_into(const double* g, uint32_t dim, float* out) {
    double n2 = 0;
    for (uint32_t d = 0; d < dim; ++d) n2 += g[d] * g[d];
    double inv = n2 > 0 ? 1.0 / std::sqrt(n2) : 0.0;
    for (uint32_t d = 0; d < dim; ++d) out[d] = float(g[d] * inv);
}

struct IvfState {
    unsigned t = 0;
    uint64_t K = 0;
    std::vector<uint64_t> bounds;  // t + 1 passage boundaries
    std::vector<uint32_t> counts;  // t x K
};

}  // namespace

extern "C" {

void synth_centroids(uint64_t K, uint32_t dim, uint64_t seed, float* out, int threads) {
    parallel_range(K, threads, [&](uint64_t b, uint64_t e, unsigned) {
        std::vector<double> g(dim);
        for (uint64_t c = b; c < e; ++c) {
            Rng r(stream_seed(seed, c));
            for (uint32_t d = 0; d < dim; ++d) g[d] = r.gauss();
            normalize_into(g.data(), dim, out + c * dim);
        }
    });
}

// Streams are keyed by the GLOBAL passage id (pid_base + p), so a passage-range
// shard generated on its own is byte-identical to the same range of the full index.
void synth_doclens(uint64_t N, uint64_t pid_base, uint32_t min_len, uint32_t max_len, uint64_t seed,
                   uint32_t* out, int threads) {
    parallel_range(N, threads, [&](uint64_t b, uint64_t e, unsigned) {
        for (uint64_t p = b; p < e; ++p) {
            Rng r(stream_seed(seed, pid_base + p));
            out[p] = min_len + uint32_t(r.below(uint64_t(max_len - min_len) + 1));
        }
    });
}

// offsets[N+1] = prefix sums of doclens; returns T.
uint64_t synth_offsets(const uint32_t* doclens, uint64_t N, uint64_t* offsets) {
    offsets[0] = 0;
    for (uint64_t p = 0; p < N; ++p) offsets[p + 1] = offsets[p] + doclens[p];
    return offsets[N];
}

void synth_codes(const uint32_t* doclens, const uint64_t* offsets, uint64_t N, uint64_t pid_base,
                 uint64_t K, double repeat_prob, uint64_t seed, uint32_t* codes, int threads) {
    parallel_range(N, threads, [&](uint64_t b, uint64_t e, unsigned) {
        for (uint64_t p = b; p < e; ++p) {
            Rng r(stream_seed(seed, pid_base + p));
            uint32_t* c = codes + offsets[p];
            for (uint32_t t = 0; t < doclens[p]; ++t) {
                if (t > 0 && r.unit() < repeat_prob)
                    c[t] = c[r.below(t)];
                else
                    c[t] = uint32_t(r.below(K));
            }
        }
    });
}

// One stream per passage covers all of its tokens' packed residual bytes.
void synth_residuals(const uint64_t* offsets, uint64_t N, uint64_t pid_base, uint64_t bytes_per_token,
                     uint64_t seed, uint8_t* out, int threads) {
    parallel_range(N, threads, [&](uint64_t b, uint64_t e, unsigned) {
        for (uint64_t p = b; p < e; ++p) {
            Rng r(stream_seed(seed, pid_base + p));
            uint8_t* o = out + offsets[p] * bytes_per_token;
            const uint64_t n = (offsets[p + 1] - offsets[p]) * bytes_per_token;
            uint64_t i = 0;
            for (; i + 8 <= n; i += 8) {
                const uint64_t v = r.next();
                std::memcpy(o + i, &v, 8);  // little-endian host
            }
            if (i < n) {
                const uint64_t v = r.next();
                for (uint64_t j = 0; i + j < n; ++j) o[i + j] = uint8_t(v >> (8 * j));
            }
        }
    });
}

// Phase 1 of the IVF build: per-thread per-centroid posting counts with
// per-passage dedup, then ivf_offsets (K+1).  Returns an opaque state for
// synth_ivf_fill (which frees it).
void* synth_ivf_count(const uint32_t* codes, const uint64_t* offsets, uint64_t N, uint64_t K,
                      uint64_t* ivf_offsets, int threads) {
    auto* st = new IvfState();
    st->t = std::min<uint64_t>(nthreads(threads), std::max<uint64_t>(N, 1));
    st->K = K;
    st->bounds.resize(st->t + 1);
    uint64_t chunk = (N + st->t - 1) / st->t;
    for (unsigned w = 0; w <= st->t; ++w) st->bounds[w] = std::min<uint64_t>(N, w * chunk);
    st->counts.assign(uint64_t(st->t) * K, 0);
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < st->t; ++w)
        pool.emplace_back([st, w, codes, offsets, K] {
            std::vector<uint32_t> seen(K, UINT32_MAX);
            uint32_t* cnt = st->counts.data() + uint64_t(w) * K;
            for (uint64_t p = st->bounds[w]; p < st->bounds[w + 1]; ++p)
                for (uint64_t t = offsets[p]; t < offsets[p + 1]; ++t) {
                    uint32_t c = codes[t];
                    if (seen[c] != uint32_t(p)) {
                        seen[c] = uint32_t(p);
                        cnt[c]++;
                    }
                }
        });
    for (auto& th : pool) th.join();
    ivf_offsets[0] = 0;
    for (uint64_t c = 0; c < K; ++c) {
        uint64_t s = 0;
        for (unsigned w = 0; w < st->t; ++w) s += st->counts[uint64_t(w) * K + c];
        ivf_offsets[c + 1] = ivf_offsets[c] + s;
    }
    return st;
}

// Phase 2: fill postings; each thread owns a passage range and writes at its
// own per-centroid cursor, so every slice comes out ascending and unique.
void synth_ivf_fill(void* state, const uint32_t* codes, const uint64_t* offsets,
                    const uint64_t* ivf_offsets, uint32_t* postings) {
    auto* st = static_cast<IvfState*>(state);
    const uint64_t K = st->K;
    // cursor[w][c] = ivf_offsets[c] + sum_{v<w} counts[v][c]  (in place)
    for (uint64_t c = 0; c < K; ++c) {
        uint64_t run = ivf_offsets[c];
        for (unsigned w = 0; w < st->t; ++w) {
            uint32_t n = st->counts[uint64_t(w) * K + c];
            st->counts[uint64_t(w) * K + c] = uint32_t(run - ivf_offsets[c]);
            run += n;
        }
    }
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < st->t; ++w)
        pool.emplace_back([st, w, codes, offsets, ivf_offsets, postings, K] {
            std::vector<uint32_t> seen(K, UINT32_MAX);
            uint32_t* cur = st->counts.data() + uint64_t(w) * K;
            for (uint64_t p = st->bounds[w]; p < st->bounds[w + 1]; ++p)
                for (uint64_t t = offsets[p]; t < offsets[p + 1]; ++t) {
                    uint32_t c = codes[t];
                    if (seen[c] != uint32_t(p)) {
                        seen[c] = uint32_t(p);
                        postings[ivf_offsets[c] + cur[c]++] = uint32_t(p);
                    }
                }
        });
    for (auto& th : pool) th.join();
    delete st;
}

// Fixed quantizer.  b=2 is the trained cfg1 quantizer; b=1
// and b=4 are symmetric stand-ins that satisfy validate_quantizer
// (residual_codec.cpp:15-40).
int synth_quantizer(uint32_t nbits, float* cutoffs, float* weights) {
    if (nbits == 1) {
        cutoffs[0] = 0.0f;
        weights[0] = -0.06f;
        weights[1] = 0.06f;
    } else if (nbits == 2) {
        const float c[3] = {-0.064f, 0.0f, 0.064f};
        const float w[4] = {-0.122f, -0.031f, 0.031f, 0.122f};
        std::memcpy(cutoffs, c, sizeof c);
        std::memcpy(weights, w, sizeof w);
    } else if (nbits == 4) {
        for (int i = 0; i < 15; ++i) cutoffs[i] = 0.02f * float(i - 7);
        weights[0] = -0.16f;
        for (int i = 1; i < 15; ++i) weights[i] = 0.5f * (cutoffs[i - 1] + cutoffs[i]);
        weights[15] = 0.16f;
    } else {
        return 4;  // PackingUnsupported + 1
    }
    return 0;
}

// Query j: stream (seed, j).  Each token picks a random passage with at least
// one token and a random token of it, reconstructs it as the reference does
// (residual_codec.cpp:97-132, float adds), adds N(0, noise^2) per dimension
// and renormalises.
void synth_queries(const float* centroids, uint32_t dim, const uint32_t* codes,
                   const uint8_t* residuals, uint32_t nbits, const float* weights,
                   const uint32_t* doclens, const uint64_t* offsets, uint64_t N, uint64_t nq,
                   uint32_t qlen, double noise, uint64_t seed, float* out) {
    const uint64_t bpt = uint64_t(nbits) * dim / 8;
    const uint32_t per = 8 / nbits, mask = (1u << nbits) - 1;
    std::vector<float> v(dim);
    std::vector<double> g(dim);
    for (uint64_t j = 0; j < nq; ++j) {
        Rng r(stream_seed(seed, j));
        for (uint32_t i = 0; i < qlen; ++i) {
            uint64_t p;
            do p = r.below(N); while (doclens[p] == 0);
            uint64_t t = offsets[p] + r.below(doclens[p]);
            const float* c = centroids + uint64_t(codes[t]) * dim;
            const uint8_t* bytes = residuals + t * bpt;
            for (uint32_t d = 0; d < dim; ++d) {
                uint32_t idx = (bytes[d / per] >> (nbits * (d % per))) & mask;
                v[d] = c[d] + weights[idx];
            }
            double n2 = 0;
            for (uint32_t d = 0; d < dim; ++d) n2 += double(v[d]) * double(v[d]);
            double inv = 1.0 / std::sqrt(n2);
            for (uint32_t d = 0; d < dim; ++d) g[d] = double(v[d]) * inv + noise * r.gauss();
            normalize_into(g.data(), dim, out + (j * qlen + i) * dim);
        }
    }
}

}  // extern "C"
