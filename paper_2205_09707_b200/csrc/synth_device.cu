// synth_device.cu — the synthetic index recipe (the same
// counter-keyed SplitMix64 streams as csrc/synth/synth.cpp) generated
// directly in HBM, for corpora too large to stage through host memory
// (BASELINE configs[4]: 140M passages / ~10B embeddings, 8 shards of ~45 GB).
//
//   centroids  thread per centroid: K rows of normalize(N(0, I_d))
//   doclens    thread per passage (stream keyed by the GLOBAL passage id)
//   offsets    one device scan
//   codes      thread per passage (repeat an earlier code of the passage with
//              probability `repeat`, else uniform over [0, K))
//   residuals  warp per passage: draw i of a SplitMix64 stream is
//              mix(seed + (i + 1) golden), so the 8-byte words are written
//              in parallel and coalesced
//   IVF        distinct (code, passage) keys with the passage's token count of
//              that code (build_inverted_list semantics, indexer.cpp:149-195),
//              one radix sort -> postings, multiplicities, offsets
//   inv norms  token_inv_norms (rank128.cu)
// Integer arrays are bit-identical to the host generator; centroids agree to
// the last bit except where the device and host libm round log/sin/cos
// differently (tests/test_gpu_synth.py bounds it).  Fixture infrastructure for
// the benchmark, not on the search path.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "device.cuh"
#include "engine.hpp"

namespace plaid {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct DRng {
    uint64_t s;
    double spare = 0;
    bool have = false;
    __device__ explicit DRng(uint64_t seed) : s(seed) {}
    __device__ uint64_t next() { return mix64(s += kGolden); }
    __device__ double unit() { return (double(next() >> 11) + 0.5) * 0x1.0p-53; }
    __device__ uint64_t below(uint64_t bound) { return bound ? next() % bound : 0; }
    __device__ double gauss() {
        if (have) {
            have = false;
            return spare;
        }
        const double u1 = unit(), u2 = unit();
        const double r = sqrt(-2.0 * log(u1));
        const double th = 6.283185307179586476925286766559 * u2;
        spare = r * sin(th);
        have = true;
        return r * cos(th);
    }
};

__device__ __forceinline__ uint64_t stream_seed(uint64_t a, uint64_t b) {
    return mix64((a ^ (kGolden + (b << 6) + (b >> 2))) + kGolden);
}

__global__ void synth_centroids_kernel(uint64_t K, uint32_t dim, uint64_t seed, float* __restrict__ out) {
    for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < K; c += uint64_t(gridDim.x) * blockDim.x) {
        DRng r(stream_seed(seed, c));
        double g[256];
        double n2 = 0;
        for (uint32_t d = 0; d < dim; ++d) {
            g[d] = r.gauss();
            n2 += g[d] * g[d];
        }
        const double inv = n2 > 0 ? 1.0 / sqrt(n2) : 0.0;
        for (uint32_t d = 0; d < dim; ++d) out[c * dim + d] = float(g[d] * inv);
    }
}

__global__ void synth_doclens_kernel(uint64_t N, uint64_t pid_base, uint32_t lo, uint32_t hi, uint64_t seed,
                                     uint32_t* __restrict__ out) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < N; p += uint64_t(gridDim.x) * blockDim.x) {
        DRng r(stream_seed(seed, pid_base + p));
        out[p] = lo + uint32_t(r.below(uint64_t(hi - lo) + 1));
    }
}

__global__ void synth_codes_kernel(const uint32_t* __restrict__ doclens, const uint64_t* __restrict__ offsets,
                                   uint64_t N, uint64_t pid_base, uint64_t K, double repeat, uint64_t seed,
                                   uint32_t* __restrict__ codes) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < N; p += uint64_t(gridDim.x) * blockDim.x) {
        DRng r(stream_seed(seed, pid_base + p));
        uint32_t* c = codes + offsets[p];
        const uint32_t len = doclens[p];
        for (uint32_t t = 0; t < len; ++t) c[t] = (t > 0 && r.unit() < repeat) ? c[r.below(t)] : uint32_t(r.below(K));
    }
}

// warp per passage: word i of the passage's residual bytes = draw i + 1
__global__ void synth_residuals_kernel(const uint64_t* __restrict__ offsets, uint64_t N, uint64_t pid_base,
                                       uint32_t bpt, uint64_t seed, uint8_t* __restrict__ out) {
    const uint32_t lane = dev::lane_id();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t p = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); p < N; p += warps) {
        const uint64_t s0 = stream_seed(seed, pid_base + p);
        const uint64_t b = offsets[p] * bpt, n = (offsets[p + 1] - offsets[p]) * bpt;  // bytes, multiple of 8
        uint64_t* o = reinterpret_cast<uint64_t*>(out + b);
        for (uint64_t i = lane; i < n / 8; i += 32) o[i] = mix64(s0 + (i + 1) * kGolden);
    }
}

// Warp per passage: its distinct codes as (code << 32 | pid) keys with the
// passage's count of that code (saturated at 255) and per-centroid counts.
__global__ void synth_postings_kernel(const uint32_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                                      uint64_t N, unsigned long long* __restrict__ nkeys,
                                      unsigned long long* __restrict__ keys, uint32_t* __restrict__ mult,
                                      unsigned long long* __restrict__ counts) {
    const uint32_t lane = dev::lane_id();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t p = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); p < N; p += warps) {
        const uint64_t b = offsets[p], e = offsets[p + 1];
        for (uint64_t t0 = b; t0 < e; t0 += 32) {
            const uint64_t t = t0 + lane;
            const uint32_t c = t < e ? codes[t] : 0xFFFFFFFFu;
            bool first = t < e;
            uint32_t m = 0;
            if (first) {
                for (uint64_t u = b; u < e; ++u) {
                    const uint32_t x = codes[u];
                    if (x == c) {
                        if (u < t) {
                            first = false;
                            break;
                        }
                        ++m;
                    }
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, first);
            unsigned long long base = 0;
            if (lane == 0 && bal) base = atomicAdd(nkeys, (unsigned long long)__popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (first) {
                const uint64_t slot = base + __popc(bal & ((1u << lane) - 1));
                keys[slot] = (uint64_t(c) << 32) | uint64_t(p);
                mult[slot] = m < 255 ? m : 255;
                atomicAdd(counts + c, 1ull);
            }
        }
    }
}

__global__ void synth_split_kernel(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ mult,
                                   uint64_t n, uint32_t* __restrict__ post, uint8_t* __restrict__ mult8) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        post[i] = uint32_t(keys[i]);
        mult8[i] = uint8_t(mult[i]);
    }
}

__global__ void widen_kernel(const uint32_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

// Queries (stream (seed, j), thread per query): each token reconstructs a
// random token of a random non-empty passage (residual_codec.cpp:97-132, fp32
// adds), adds N(0, noise^2) per dim and renormalises.
__global__ void synth_queries_kernel(const float* __restrict__ C, uint32_t dim, const uint32_t* __restrict__ codes,
                                     const uint8_t* __restrict__ residuals, uint32_t nbits, const float* __restrict__ W,
                                     const uint32_t* __restrict__ doclens, const uint64_t* __restrict__ offsets,
                                     uint64_t N, uint64_t nq, uint32_t qlen, double noise, uint64_t seed,
                                     float* __restrict__ out) {
    const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (j >= nq) return;
    const uint64_t bpt = uint64_t(nbits) * dim / 8;
    const uint32_t per = 8 / nbits, mask = (1u << nbits) - 1;
    DRng r(stream_seed(seed, j));
    float v[256];
    double g[256];
    for (uint32_t i = 0; i < qlen; ++i) {
        uint64_t p;
        do p = r.below(N);
        while (doclens[p] == 0);
        const uint64_t t = offsets[p] + r.below(doclens[p]);
        const float* c = C + uint64_t(codes[t]) * dim;
        const uint8_t* bytes = residuals + t * bpt;
        for (uint32_t d = 0; d < dim; ++d) v[d] = __fadd_rn(c[d], W[(bytes[d / per] >> (nbits * (d % per))) & mask]);
        double n2 = 0;
        for (uint32_t d = 0; d < dim; ++d) n2 += double(v[d]) * double(v[d]);
        const double inv = 1.0 / sqrt(n2);
        for (uint32_t d = 0; d < dim; ++d) g[d] = double(v[d]) * inv + noise * r.gauss();
        double m2 = 0;
        for (uint32_t d = 0; d < dim; ++d) m2 += g[d] * g[d];
        const double minv = m2 > 0 ? 1.0 / sqrt(m2) : 0.0;
        for (uint32_t d = 0; d < dim; ++d) out[(j * qlen + i) * dim + d] = float(g[d] * minv);
    }
}

uint32_t grid_of(uint64_t n, uint32_t threads, uint32_t cap) {
    const uint64_t b = (n + threads - 1) / threads;
    return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

template <typename T>
struct Tmp {
    T* p = nullptr;
    explicit Tmp(uint64_t n) { PLAID_CUDA(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T))); }
    ~Tmp() { cudaFree(p); }
    Tmp(const Tmp&) = delete;
    Tmp& operator=(const Tmp&) = delete;
};

// the fixed quantizer of SURVEY.md §8d (synth.cpp synth_quantizer)
void quantizer(uint32_t nbits, float* cut, float* w) {
    if (nbits == 1) {
        cut[0] = 0.0f;
        w[0] = -0.06f;
        w[1] = 0.06f;
    } else if (nbits == 2) {
        const float c[3] = {-0.064f, 0.0f, 0.064f};
        const float ww[4] = {-0.122f, -0.031f, 0.031f, 0.122f};
        std::memcpy(cut, c, sizeof c);
        std::memcpy(w, ww, sizeof ww);
    } else {
        for (int i = 0; i < 15; ++i) cut[i] = 0.02f * float(i - 7);
        w[0] = -0.16f;
        for (int i = 1; i < 15; ++i) w[i] = 0.5f * (cut[i - 1] + cut[i]);
        w[15] = 0.16f;
    }
}

}  // namespace

DeviceIndex::DeviceIndex(const SynthSpec& sp, int device) : device_(device), pid_base_(sp.pid_base) {
    if (sp.nbits != 1 && sp.nbits != 2 && sp.nbits != 4) fail(PLAID_PACKING_UNSUPPORTED, "nbits must be one of {1,2,4}");
    if (sp.dim == 0 || sp.dim > 256 || (sp.dim * sp.nbits) % 64)
        fail(PLAID_UNSUPPORTED, "synthetic index: dim <= 256 with dim * nbits a multiple of 64");
    if (sp.num_passages == 0 || sp.num_passages > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "passages in [1, 2^32)");
    if (sp.num_centroids == 0 || sp.num_centroids > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "centroids in [1, 2^32)");
    DeviceGuard g(device);
    const uint64_t N = sp.num_passages, K = sp.num_centroids;
    const uint32_t dim = sp.dim, nbits = sp.nbits, bpt = dim * nbits / 8;
    const uint32_t lo = sp.mean_len > sp.spread ? sp.mean_len - sp.spread : 1, hi = sp.mean_len + sp.spread;
    cudaStream_t st = nullptr;
    auto alloc = [&](uint64_t bytes) {
        void* p = nullptr;
        PLAID_CUDA(cudaMalloc(&p, std::max<uint64_t>(bytes, 1)));
        allocs_.push_back(p);
        bytes_ += bytes;
        return p;
    };
    try {
        view_.dim = dim;
        view_.nbits = nbits;
        view_.K = K;
        view_.N = N;
        float cut[16] = {}, w[16] = {};
        quantizer(nbits, cut, w);
        for (uint32_t i = 0; i < (1u << nbits); ++i) view_.weights[i] = w[i];
        for (uint32_t i = 0; i + 1 < (1u << nbits); ++i) cutoffs_[i] = cut[i];
        float* C = static_cast<float*>(alloc(K * dim * 4));
        synth_centroids_kernel<<<grid_of(K, 128, 148 * 64), 128, 0, st>>>(K, dim, 11 + sp.seed, C);
        uint32_t* dl = static_cast<uint32_t*>(alloc(N * 4));
        synth_doclens_kernel<<<grid_of(N, 256, 148 * 64), 256, 0, st>>>(N, sp.pid_base, lo, hi, 5 + sp.seed, dl);
        PLAID_CUDA(cudaGetLastError());
        uint64_t* off = static_cast<uint64_t*>(alloc((N + 1) * 8));
        {
            Tmp<uint64_t> wide(N + 1);
            widen_kernel<<<grid_of(N, 256, 148 * 64), 256, 0, st>>>(dl, N, wide.p);
            PLAID_CUDA(cudaMemsetAsync(wide.p + N, 0, 8, st));
            size_t tb = 0;
            PLAID_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, wide.p, off, N + 1, st));
            Tmp<uint8_t> t(tb);
            PLAID_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, wide.p, off, N + 1, st));
            PLAID_CUDA(cudaStreamSynchronize(st));
        }
        uint64_t T = 0;
        PLAID_CUDA(cudaMemcpy(&T, off + N, 8, cudaMemcpyDeviceToHost));
        view_.T = T;
        uint32_t* codes = static_cast<uint32_t*>(alloc(T * 4));
        synth_codes_kernel<<<grid_of(N, 128, 148 * 64), 128, 0, st>>>(dl, off, N, sp.pid_base, K, sp.repeat, 99 + sp.seed,
                                                                     codes);
        uint8_t* res = static_cast<uint8_t*>(alloc(T * bpt));
        synth_residuals_kernel<<<grid_of(N * 32, 256, 148 * 32), 256, 0, st>>>(off, N, sp.pid_base, bpt, 7 + sp.seed,
                                                                               res);
        PLAID_CUDA(cudaGetLastError());
        // IVF: distinct (code, pid) keys + multiplicities, one radix sort
        Tmp<unsigned long long> counts(K + 1), nk(1);
        PLAID_CUDA(cudaMemsetAsync(counts.p, 0, (K + 1) * 8, st));
        PLAID_CUDA(cudaMemsetAsync(nk.p, 0, 8, st));
        unsigned long long P = 0;
        uint64_t* ivo = static_cast<uint64_t*>(alloc((K + 1) * 8));
        uint32_t* post = nullptr;
        uint8_t* mult8 = nullptr;
        {
            Tmp<unsigned long long> keys(T), skeys(T);
            Tmp<uint32_t> mult(T), smult(T);
            synth_postings_kernel<<<grid_of(N * 32, 256, 148 * 16), 256, 0, st>>>(codes, off, N, nk.p, keys.p, mult.p,
                                                                                  counts.p);
            PLAID_CUDA(cudaGetLastError());
            PLAID_CUDA(cudaMemcpy(&P, nk.p, 8, cudaMemcpyDeviceToHost));
            int end_bit = 32;
            while (end_bit < 64 && ((K - 1) >> (end_bit - 32))) ++end_bit;
            size_t tb = 0;
            PLAID_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, mult.p, smult.p, P, 0, end_bit, st));
            {
                Tmp<uint8_t> t(tb);
                PLAID_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, keys.p, skeys.p, mult.p, smult.p, P, 0, end_bit, st));
                PLAID_CUDA(cudaStreamSynchronize(st));
            }
            post = static_cast<uint32_t*>(alloc(P * 4));
            mult8 = static_cast<uint8_t*>(alloc(P));
            synth_split_kernel<<<grid_of(P, 256, 148 * 16), 256, 0, st>>>(skeys.p, smult.p, P, post, mult8);
            size_t sb = 0;
            PLAID_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, counts.p, ivo, K + 1, st));
            Tmp<uint8_t> t2(sb);
            PLAID_CUDA(cub::DeviceScan::ExclusiveSum(t2.p, sb, counts.p, ivo, K + 1, st));
            PLAID_CUDA(cudaStreamSynchronize(st));
        }
        view_.P = P;
        view_.centroids = C;
        view_.codes = codes;
        view_.residuals = res;
        view_.doclens = dl;
        view_.offsets = off;
        view_.ivf_offsets = ivo;
        view_.ivf_postings = post;
        view_.ivf_mult = mult8;
        h_doclens_.resize(N);
        PLAID_CUDA(cudaMemcpy(h_doclens_.data(), dl, N * 4, cudaMemcpyDeviceToHost));
        {
            std::vector<uint64_t> h_ivo(K + 1);
            PLAID_CUDA(cudaMemcpy(h_ivo.data(), ivo, (K + 1) * 8, cudaMemcpyDeviceToHost));
            set_list_bounds(h_ivo.data());
        }
        for (uint32_t x : h_doclens_) max_doclen_ = std::max(max_doclen_, x);
        view_.max_doclen = max_doclen_;
        if (dim == 128 && T) {
            float* inv = static_cast<float*>(alloc(T * 4));
            launch::token_inv_norms(view_, inv, st);
            view_.tok_inv = inv;
        }
        build_range_table(st);
        PLAID_CUDA(cudaStreamSynchronize(st));
        PLAID_CUDA(cudaGetLastError());
    } catch (...) {
        for (void* p : allocs_) cudaFree(p);
        allocs_.clear();
        throw;
    }
}

void DeviceIndex::synth_queries(uint64_t nq, uint32_t qlen, double noise, uint64_t seed, float* out_host) const {
    if (qlen == 0 || qlen > 32) fail(PLAID_UNSUPPORTED, "query length must be in [1, 32]");
    DeviceGuard g(device_);
    const IndexView& v = view_;
    Tmp<float> d_out(nq * qlen * v.dim), d_w(16);
    PLAID_CUDA(cudaMemcpy(d_w.p, v.weights, sizeof v.weights, cudaMemcpyHostToDevice));
    synth_queries_kernel<<<uint32_t((nq + 63) / 64), 64>>>(v.centroids, v.dim, v.codes, v.residuals, v.nbits, d_w.p,
                                                          v.doclens, v.offsets, v.N, nq, qlen, noise, seed, d_out.p);
    PLAID_CUDA(cudaGetLastError());
    PLAID_CUDA(cudaMemcpy(out_host, d_out.p, nq * qlen * v.dim * 4, cudaMemcpyDeviceToHost));
}

void DeviceIndex::export_host(float* centroids, uint32_t* codes, uint8_t* residuals, uint32_t* doclens,
                              uint64_t* ivf_offsets, uint32_t* ivf_postings, float* cutoffs, float* weights) const {
    DeviceGuard g(device_);
    const IndexView& v = view_;
    const uint64_t bpt = uint64_t(v.nbits) * v.dim / 8;
    if (centroids) PLAID_CUDA(cudaMemcpy(centroids, v.centroids, v.K * v.dim * 4, cudaMemcpyDeviceToHost));
    if (codes) PLAID_CUDA(cudaMemcpy(codes, v.codes, v.T * 4, cudaMemcpyDeviceToHost));
    if (residuals) PLAID_CUDA(cudaMemcpy(residuals, v.residuals, v.T * bpt, cudaMemcpyDeviceToHost));
    if (doclens) std::memcpy(doclens, h_doclens_.data(), v.N * 4);
    if (ivf_offsets) PLAID_CUDA(cudaMemcpy(ivf_offsets, v.ivf_offsets, (v.K + 1) * 8, cudaMemcpyDeviceToHost));
    if (ivf_postings) PLAID_CUDA(cudaMemcpy(ivf_postings, v.ivf_postings, v.P * 4, cudaMemcpyDeviceToHost));
    if (cutoffs) std::memcpy(cutoffs, cutoffs_, ((1u << v.nbits) - 1) * 4);
    if (weights) std::memcpy(weights, v.weights, (1u << v.nbits) * 4);
}

}  // namespace plaid
