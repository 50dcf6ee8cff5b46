/*
 * synth_oracle.c — TEST INFRASTRUCTURE: an independent C restatement of the
 * synthetic index recipe of SURVEY.md §8d / Appendix A.1, so the reference
 * arm of bench.py (and the tests) can build the benchmark inputs without
 * loading any of the product's libraries.
 *
 * The recipe (every stream a counter-keyed SplitMix64, the algorithm of the
 * reference's rng.hpp:11-56):
 *   centroids  K rows of normalize(N(0, I_d)), stream (seed_c, c)
 *   doclens    min_len + U{0 .. max_len - min_len}, stream (seed_d, global pid)
 *   codes      per passage, token t > 0 repeats an earlier code of the same
 *              passage with probability `repeat`, else uniform over [0, K),
 *              stream (seed_k, global pid)
 *   residuals  uniform random bytes, 8 per draw LSB first, stream (seed_r, pid)
 *   queries    token = normalize(reconstruct(random token) + N(0, noise^2))
 *              (reconstruct as residual_codec.cpp:97-132, float adds)
 * The IVF is left to the reference's own build_inverted_list
 * (indexer.cpp:149-195, via oracle/_ref) or to the caller.
 *
 * tests/test_synth.py checks that these bytes equal the product generator's
 * (paper_2205_09707_b200/csrc/synth), which pins the benchmark inputs.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef struct {
    uint64_t s;
    double spare;
    int have;
} osyn_rng;

static uint64_t rng_next(osyn_rng* r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double rng_unit(osyn_rng* r) { return ((double)(rng_next(r) >> 11) + 0.5) * 0x1.0p-53; }

static uint64_t rng_below(osyn_rng* r, uint64_t bound) { return bound ? rng_next(r) % bound : 0; }

/* Box-Muller pair: cos branch first, the sin branch cached for the next call */
static double rng_gauss(osyn_rng* r) {
    if (r->have) {
        r->have = 0;
        return r->spare;
    }
    const double u1 = rng_unit(r), u2 = rng_unit(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double th = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(th);
    r->have = 1;
    return rad * cos(th);
}

static osyn_rng rng_make(uint64_t seed) {
    osyn_rng r = {seed, 0.0, 0};
    return r;
}

/* the seed of stream (a, b): first draw of a generator keyed by a and b */
static uint64_t stream_seed(uint64_t a, uint64_t b) {
    osyn_rng r = rng_make(a ^ (0x9E3779B97F4A7C15ULL + (b << 6) + (b >> 2)));
    return rng_next(&r);
}

static void normalize_into(const double* g, uint32_t dim, float* out) {
    double n2 = 0;
    for (uint32_t d = 0; d < dim; ++d) n2 += g[d] * g[d];
    const double inv = n2 > 0 ? 1.0 / sqrt(n2) : 0.0;
    for (uint32_t d = 0; d < dim; ++d) out[d] = (float)(g[d] * inv);
}

/* ---- a tiny parallel-for over [0, n) -------------------------------------------- */
typedef void (*range_fn)(void* ctx, uint64_t b, uint64_t e);
typedef struct {
    range_fn fn;
    void* ctx;
    uint64_t b, e;
} range_job;

static void* range_thread(void* a) {
    range_job* j = (range_job*)a;
    j->fn(j->ctx, j->b, j->e);
    return NULL;
}

static void parallel_for(uint64_t n, int threads, range_fn fn, void* ctx) {
    long t = threads > 0 ? threads : sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if ((uint64_t)t > n) t = n ? (long)n : 1;
    if (t > 256) t = 256;
    pthread_t th[256];
    range_job jobs[256];
    const uint64_t chunk = (n + (uint64_t)t - 1) / (uint64_t)t;
    long started = 0;
    for (long w = 0; w < t; ++w) {
        const uint64_t b = (uint64_t)w * chunk, e = b + chunk < n ? b + chunk : n;
        if (b >= e) break;
        jobs[w] = (range_job){fn, ctx, b, e};
        if (t == 1) {
            fn(ctx, b, e);
            return;
        }
        pthread_create(&th[w], NULL, range_thread, &jobs[w]);
        ++started;
    }
    for (long w = 0; w < started; ++w) pthread_join(th[w], NULL);
}

/* ---- centroids ---------------------------------------------------------------------- */
typedef struct {
    uint32_t dim;
    uint64_t seed;
    float* out;
} cent_ctx;

static void cent_range(void* c, uint64_t b, uint64_t e) {
    cent_ctx* x = (cent_ctx*)c;
    double* g = (double*)malloc(sizeof(double) * x->dim);
    for (uint64_t k = b; k < e; ++k) {
        osyn_rng r = rng_make(stream_seed(x->seed, k));
        for (uint32_t d = 0; d < x->dim; ++d) g[d] = rng_gauss(&r);
        normalize_into(g, x->dim, x->out + k * x->dim);
    }
    free(g);
}

void osyn_centroids(uint64_t K, uint32_t dim, uint64_t seed, float* out, int threads) {
    cent_ctx c = {dim, seed, out};
    parallel_for(K, threads, cent_range, &c);
}

/* ---- doclens (stream keyed by the GLOBAL passage id) ------------------------------- */
typedef struct {
    uint64_t pid_base, seed;
    uint32_t lo, hi;
    uint32_t* out;
} len_ctx;

static void len_range(void* c, uint64_t b, uint64_t e) {
    len_ctx* x = (len_ctx*)c;
    for (uint64_t p = b; p < e; ++p) {
        osyn_rng r = rng_make(stream_seed(x->seed, x->pid_base + p));
        x->out[p] = x->lo + (uint32_t)rng_below(&r, (uint64_t)(x->hi - x->lo) + 1);
    }
}

void osyn_doclens(uint64_t N, uint64_t pid_base, uint32_t min_len, uint32_t max_len, uint64_t seed, uint32_t* out,
                  int threads) {
    len_ctx c = {pid_base, seed, min_len, max_len, out};
    parallel_for(N, threads, len_range, &c);
}

/* ---- codes -------------------------------------------------------------------------- */
typedef struct {
    const uint32_t* doclens;
    const uint64_t* offsets;
    uint64_t pid_base, K, seed;
    double repeat;
    uint32_t* codes;
} code_ctx;

static void code_range(void* c, uint64_t b, uint64_t e) {
    code_ctx* x = (code_ctx*)c;
    for (uint64_t p = b; p < e; ++p) {
        osyn_rng r = rng_make(stream_seed(x->seed, x->pid_base + p));
        uint32_t* out = x->codes + x->offsets[p];
        for (uint32_t t = 0; t < x->doclens[p]; ++t) {
            if (t > 0 && rng_unit(&r) < x->repeat)
                out[t] = out[rng_below(&r, t)];
            else
                out[t] = (uint32_t)rng_below(&r, x->K);
        }
    }
}

void osyn_codes(const uint32_t* doclens, const uint64_t* offsets, uint64_t N, uint64_t pid_base, uint64_t K,
                double repeat, uint64_t seed, uint32_t* codes, int threads) {
    code_ctx c = {doclens, offsets, pid_base, K, seed, repeat, codes};
    parallel_for(N, threads, code_range, &c);
}

/* ---- residual bytes: one stream per passage, 8 bytes per draw, LSB first ----------- */
typedef struct {
    const uint64_t* offsets;
    uint64_t pid_base, bpt, seed;
    uint8_t* out;
} res_ctx;

static void res_range(void* c, uint64_t b, uint64_t e) {
    res_ctx* x = (res_ctx*)c;
    for (uint64_t p = b; p < e; ++p) {
        osyn_rng r = rng_make(stream_seed(x->seed, x->pid_base + p));
        uint8_t* o = x->out + x->offsets[p] * x->bpt;
        const uint64_t n = (x->offsets[p + 1] - x->offsets[p]) * x->bpt;
        for (uint64_t i = 0; i < n; i += 8) {
            const uint64_t v = rng_next(&r);
            for (uint64_t j = 0; j < 8 && i + j < n; ++j) o[i + j] = (uint8_t)(v >> (8 * j));
        }
    }
}

void osyn_residuals(const uint64_t* offsets, uint64_t N, uint64_t pid_base, uint64_t bytes_per_token, uint64_t seed,
                    uint8_t* out, int threads) {
    res_ctx c = {offsets, pid_base, bytes_per_token, seed, out};
    parallel_for(N, threads, res_range, &c);
}

/* ---- the fixed quantizer of SURVEY.md §8d ------------------------------------------ */
int osyn_quantizer(uint32_t nbits, float* cutoffs, float* weights) {
    if (nbits == 1) {
        cutoffs[0] = 0.0f;
        weights[0] = -0.06f;
        weights[1] = 0.06f;
    } else if (nbits == 2) {
        const float c[3] = {-0.064f, 0.0f, 0.064f};
        const float w[4] = {-0.122f, -0.031f, 0.031f, 0.122f};
        memcpy(cutoffs, c, sizeof c);
        memcpy(weights, w, sizeof w);
    } else if (nbits == 4) {
        for (int i = 0; i < 15; ++i) cutoffs[i] = 0.02f * (float)(i - 7);
        weights[0] = -0.16f;
        for (int i = 1; i < 15; ++i) weights[i] = 0.5f * (cutoffs[i - 1] + cutoffs[i]);
        weights[15] = 0.16f;
    } else {
        return 4; /* PackingUnsupported + 1 */
    }
    return 0;
}

/* ---- queries: stream (seed, j) ------------------------------------------------------- */
void osyn_queries(const float* centroids, uint32_t dim, const uint32_t* codes, const uint8_t* residuals,
                  uint32_t nbits, const float* weights, const uint32_t* doclens, const uint64_t* offsets, uint64_t N,
                  uint64_t nq, uint32_t qlen, double noise, uint64_t seed, float* out) {
    const uint64_t bpt = (uint64_t)nbits * dim / 8;
    const uint32_t per = 8 / nbits, mask = (1u << nbits) - 1;
    float* v = (float*)malloc(sizeof(float) * dim);
    double* g = (double*)malloc(sizeof(double) * dim);
    for (uint64_t j = 0; j < nq; ++j) {
        osyn_rng r = rng_make(stream_seed(seed, j));
        for (uint32_t i = 0; i < qlen; ++i) {
            uint64_t p;
            do p = rng_below(&r, N);
            while (doclens[p] == 0);
            const uint64_t t = offsets[p] + rng_below(&r, doclens[p]);
            const float* c = centroids + (uint64_t)codes[t] * dim;
            const uint8_t* bytes = residuals + t * bpt;
            for (uint32_t d = 0; d < dim; ++d) {
                const uint32_t idx = (bytes[d / per] >> (nbits * (d % per))) & mask;
                v[d] = c[d] + weights[idx];
            }
            double n2 = 0;
            for (uint32_t d = 0; d < dim; ++d) n2 += (double)v[d] * (double)v[d];
            const double inv = 1.0 / sqrt(n2);
            for (uint32_t d = 0; d < dim; ++d) g[d] = (double)v[d] * inv + noise * rng_gauss(&r);
            normalize_into(g, dim, out + (j * qlen + i) * dim);
        }
    }
    free(v);
    free(g);
}
