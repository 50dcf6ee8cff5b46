// encode.cu — the encode half of index building on the GPU (SURVEY.md §8f
// rank 2): given trained centroids and quantizer, compute what
// lir::build_index (indexer.cpp:197-282) derives from them —
//   codes      assign_codes        (indexer.cpp:45-72): argmax_c dot(v, C[c]),
//              in-order fp32 dots without FMA (types.hpp:18-22), first max wins;
//   residuals  quantise + pack      (indexer.cpp:262-280, residual_codec.hpp:23-31):
//              bucket = #cutoffs <= v[d] - C[code][d], LSB-first packing;
//   IVF        build_inverted_list (indexer.cpp:149-195): per centroid the
//              sorted unique ids of the passages owning it.
// Bit-identical to the reference (tests/test_gpu_parity.py::test_encode_*).
// build_index_host (below) adds k-means and the quantizer fit (kmeans.cpp,
// indexer.cpp:74-147): their seed-driven sequential choices stay on the host
// in the reference's order, the dots and sums run on the GPU.
//
// assign_codes is the only heavy part (T x K x d multiply-adds).  Exactness
// pins it to the FP32 pipe (a rounded multiply and a rounded add per term):
// a thread owns one token (its dims read from a [d][token] shared-memory
// tile, conflict-free), a block walks the centroids in chunks of 8 staged as
// [d][8] (two broadcast LDS.128 per dim), so each dim costs 1 + 2 loads for
// 16 FP32 ops.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "device.cuh"
#include "encode.hpp"
#include "engine.hpp"

namespace plaid {
namespace {

constexpr uint32_t kTokTile = 128;  // tokens per block (one per thread)
constexpr uint32_t kCentChunk = 8;  // centroids per staged chunk

__global__ void __launch_bounds__(kTokTile)
assign_codes_kernel(const float* __restrict__ emb, uint64_t T, const float* __restrict__ C, uint32_t K, uint32_t dim,
                    uint32_t* __restrict__ codes, float* __restrict__ top_out) {
    extern __shared__ __align__(16) float sh[];
    float* vt = sh;                             // [dim][kTokTile]
    float* ct = sh + size_t(dim) * kTokTile;    // [dim][kCentChunk]
    const uint64_t t0 = uint64_t(blockIdx.x) * kTokTile;
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = tid; i < dim * kTokTile; i += kTokTile) {
        const uint32_t tok = i / dim, d = i % dim;  // coalesced global read, transposed store
        vt[d * kTokTile + tok] = t0 + tok < T ? emb[(t0 + tok) * dim + d] : 0.f;
    }
    float top = -INFINITY;
    uint32_t arg = 0;
    for (uint32_t c0 = 0; c0 < K; c0 += kCentChunk) {
        __syncthreads();
        for (uint32_t i = tid; i < dim * kCentChunk; i += kTokTile) {
            const uint32_t c = i / dim, d = i % dim;
            ct[d * kCentChunk + c] = c0 + c < K ? C[uint64_t(c0 + c) * dim + d] : 0.f;
        }
        __syncthreads();
        float acc[kCentChunk];
#pragma unroll
        for (uint32_t j = 0; j < kCentChunk; ++j) acc[j] = 0.f;
#pragma unroll 4
        for (uint32_t d = 0; d < dim; ++d) {
            const float v = vt[d * kTokTile + tid];
            const float4 a = *reinterpret_cast<const float4*>(ct + d * kCentChunk);
            const float4 b = *reinterpret_cast<const float4*>(ct + d * kCentChunk + 4);
            acc[0] = dev::madd_rn(acc[0], v, a.x);
            acc[1] = dev::madd_rn(acc[1], v, a.y);
            acc[2] = dev::madd_rn(acc[2], v, a.z);
            acc[3] = dev::madd_rn(acc[3], v, a.w);
            acc[4] = dev::madd_rn(acc[4], v, b.x);
            acc[5] = dev::madd_rn(acc[5], v, b.y);
            acc[6] = dev::madd_rn(acc[6], v, b.z);
            acc[7] = dev::madd_rn(acc[7], v, b.w);
        }
        // indexer.cpp:58-67: top = dot(v, C[0]); later centroids replace it
        // only with a strictly larger score
#pragma unroll
        for (uint32_t j = 0; j < kCentChunk; ++j) {
            if (c0 + j < K && (c0 + j == 0 || acc[j] > top)) {
                top = acc[j];
                arg = c0 + j;
            }
        }
    }
    if (t0 + tid < T) {
        codes[t0 + tid] = arg;
        if (top_out) top_out[t0 + tid] = top;  // the winning dot (k-means empty-cluster repair)
    }
}

// Thread per (token, residual byte): the byte's 8/b dims, bucket = number of
// cutoffs <= (v[d] - C[code][d]) (residual_codec.hpp:23-31), LSB first.
__global__ void quantize_pack_kernel(const float* __restrict__ emb, const float* __restrict__ C,
                                     const uint32_t* __restrict__ codes, uint64_t T, uint32_t dim, uint32_t nbits,
                                     const float* __restrict__ cutoffs, uint8_t* __restrict__ out) {
    __shared__ float cut[15];
    const uint32_t ncut = (1u << nbits) - 1;
    if (threadIdx.x < ncut) cut[threadIdx.x] = cutoffs[threadIdx.x];
    __syncthreads();
    const uint32_t per_byte = 8 / nbits, bpt = dim / per_byte;
    const uint64_t total = T * bpt;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t t = i / bpt;
        const uint32_t j = uint32_t(i % bpt);
        const float* v = emb + t * dim + j * per_byte;
        const float* c = C + uint64_t(codes[t]) * dim + j * per_byte;
        uint32_t byte = 0;
        for (uint32_t e = 0; e < per_byte; ++e) {
            const float x = __fsub_rn(v[e], c[e]);
            uint32_t b = 0;
            for (uint32_t k = 0; k < ncut; ++k) b += cut[k] <= x;
            byte |= b << (nbits * e);
        }
        out[i] = uint8_t(byte);
    }
}

// Warp per passage: its distinct codes -> (code << 32 | pid) keys (passage
// order irrelevant: a global radix sort orders them) and per-centroid counts.
__global__ void passage_postings_kernel(const uint32_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                                        uint64_t N, unsigned long long* __restrict__ nkeys,
                                        unsigned long long* __restrict__ keys, unsigned long long* __restrict__ counts) {
    const uint32_t lane = dev::lane_id();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t p = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); p < N; p += warps) {
        const uint64_t b = offsets[p], e = offsets[p + 1];
        for (uint64_t t0 = b; t0 < e; t0 += 32) {
            const uint64_t t = t0 + lane;
            const uint32_t c = t < e ? codes[t] : 0xFFFFFFFFu;
            // first occurrence in the passage?
            bool first = t < e;
            for (uint64_t u = b; u < t0 && first; ++u) first = codes[u] != c;
            for (uint32_t l = 0; l < 32; ++l) {
                const uint32_t o = __shfl_sync(0xffffffffu, c, l);
                if (l < lane && o == c) first = false;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, first);
            unsigned long long base = 0;
            if (lane == 0 && bal) base = atomicAdd(nkeys, (unsigned long long)__popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (first) {
                keys[base + __popc(bal & ((1u << lane) - 1))] = (uint64_t(c) << 32) | uint64_t(p);
                atomicAdd(counts + c, 1ull);
            }
        }
    }
}

__global__ void low_words_kernel(const unsigned long long* __restrict__ keys, uint64_t n, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = uint32_t(keys[i]);
}

template <typename T>
struct Dev {
    T* p = nullptr;
    explicit Dev(uint64_t n) { PLAID_CUDA(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T))); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

// k-means++ seeding step (kmeans.cpp:101-128): bd[j] = max(bd[j], dot(p_j, c))
// with the reference's in-order fp32 dot; init: bd[j] = dot(p_j, c).
__global__ void seed_update_kernel(const float* __restrict__ pts, uint64_t n, uint32_t dim, const float* __restrict__ c,
                                   float* __restrict__ bd, int init) {
    extern __shared__ float cs[];
    for (uint32_t i = threadIdx.x; i < dim; i += blockDim.x) cs[i] = c[i];
    __syncthreads();
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x) {
        const float* pj = pts + j * dim;
        float acc = 0.f;
        for (uint32_t d = 0; d < dim; ++d) acc = dev::madd_rn(acc, pj[d], cs[d]);
        if (init || acc > bd[j]) bd[j] = acc;
    }
}

// Lloyd mean update (kmeans.cpp:152-171): thread per (cluster, dim) sums its
// cluster's member points IN POINT ORDER in double (members = a stable
// counting sort of the assignment, so each sum is the reference's sequential
// loop restricted to one cluster); then thread per cluster: the in-order norm
// and the normalised centroid (kept when empty or degenerate).
__global__ void mean_sum_kernel(const float* __restrict__ pts, uint32_t dim, const uint32_t* __restrict__ members,
                                const uint64_t* __restrict__ moff, uint64_t k, double* __restrict__ sums) {
    const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (e >= k * dim) return;
    const uint64_t c = e / dim, i = e % dim;
    double acc = 0.0;
    for (uint64_t m = moff[c]; m < moff[c + 1]; ++m) acc += double(pts[uint64_t(members[m]) * dim + i]);
    sums[e] = acc;
}

__global__ void mean_norm_kernel(const double* __restrict__ sums, const uint64_t* __restrict__ moff, uint64_t k,
                                 uint32_t dim, float* __restrict__ C) {
    const uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (c >= k || moff[c + 1] == moff[c]) return;  // empty: keep repaired/stolen centroid
    const double* s = sums + c * dim;
    double norm_sq = 0.0;
    for (uint32_t i = 0; i < dim; ++i) norm_sq += s[i] * s[i];
    if (norm_sq <= 1e-24) return;  // degenerate mean: keep previous centroid
    const double inv = 1.0 / sqrt(norm_sq);
    for (uint32_t i = 0; i < dim; ++i) C[c * dim + i] = float(s[i] * inv);
}

uint32_t grid_cap(uint64_t n, uint32_t threads, uint32_t cap) {
    const uint64_t b = (n + threads - 1) / threads;
    return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

}  // namespace

void encode_host(const plaid_encode_desc& in, int device, uint32_t* codes, uint8_t* residuals, uint64_t* ivf_offsets,
                 uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings) {
    const uint32_t dim = in.dim, nbits = in.nbits;
    const uint64_t N = in.num_passages, K = in.num_centroids;
    // build_index's checks, in its order (indexer.cpp:199-213, types.cpp:31-47)
    std::vector<uint64_t> off(N + 1, 0);
    for (uint64_t p = 0; p < N; ++p) off[p + 1] = off[p] + in.doclens[p];
    const uint64_t T = off[N];
    if (N == 0 || T == 0) fail(PLAID_EMPTY_CORPUS, "cannot index an empty corpus");
    if (T != in.num_embeddings) fail(PLAID_LENGTH_MISMATCH, "doclens total does not match the embedding rows");
    if (nbits != 1 && nbits != 2 && nbits != 4) fail(PLAID_PACKING_UNSUPPORTED, "nbits must be one of {1,2,4}");
    if (dim == 0 || dim % (8 / nbits) != 0)
        fail(PLAID_PACKING_UNSUPPORTED, "dim " + std::to_string(dim) + " not divisible by " +
                                            std::to_string(8 / nbits) + " for nbits " + std::to_string(nbits));
    if (N > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "corpora above 2^32 passages are not supported");
    if (dim > 1024) fail(PLAID_UNSUPPORTED, "encode supports dim <= 1024");
    if (K == 0 || K > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "centroid count must be in [1, 2^32)");
    validate_query_host(in.embeddings, T, dim, dim);  // check_unit_rows: NotNormalized (types.cpp:10-19)
    DeviceGuard g(device);
    cudaStream_t st = nullptr;
    const uint32_t bpt = dim * nbits / 8;
    Dev<float> d_emb(T * dim), d_C(K * dim), d_cut(16);
    Dev<uint32_t> d_codes(T);
    Dev<uint8_t> d_res(T * bpt);
    Dev<uint64_t> d_off(N + 1);
    PLAID_CUDA(cudaMemcpy(d_emb.p, in.embeddings, T * dim * 4, cudaMemcpyHostToDevice));
    PLAID_CUDA(cudaMemcpy(d_C.p, in.centroids, K * dim * 4, cudaMemcpyHostToDevice));
    PLAID_CUDA(cudaMemcpy(d_cut.p, in.bucket_cutoffs, ((1u << nbits) - 1) * 4, cudaMemcpyHostToDevice));
    PLAID_CUDA(cudaMemcpy(d_off.p, off.data(), (N + 1) * 8, cudaMemcpyHostToDevice));

    const size_t smem = size_t(dim) * (kTokTile + kCentChunk) * sizeof(float);
    PLAID_CUDA(cudaFuncSetAttribute(assign_codes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    assign_codes_kernel<<<uint32_t((T + kTokTile - 1) / kTokTile), kTokTile, smem, st>>>(d_emb.p, T, d_C.p, uint32_t(K),
                                                                                        dim, d_codes.p, nullptr);
    PLAID_CUDA(cudaGetLastError());
    quantize_pack_kernel<<<grid_cap(T * bpt, 256, 148 * 32), 256, 0, st>>>(d_emb.p, d_C.p, d_codes.p, T, dim, nbits,
                                                                           d_cut.p, d_res.p);
    PLAID_CUDA(cudaGetLastError());

    // IVF: distinct (code, pid) keys, one radix sort, counts -> offsets
    Dev<unsigned long long> d_keys(T), d_sorted(T), d_counts(K + 1), d_n(1);
    PLAID_CUDA(cudaMemsetAsync(d_counts.p, 0, (K + 1) * 8, st));
    PLAID_CUDA(cudaMemsetAsync(d_n.p, 0, 8, st));
    passage_postings_kernel<<<grid_cap(N * 32, 256, 148 * 16), 256, 0, st>>>(d_codes.p, d_off.p, N, d_n.p, d_keys.p,
                                                                              d_counts.p);
    PLAID_CUDA(cudaGetLastError());
    unsigned long long P = 0;
    PLAID_CUDA(cudaMemcpy(&P, d_n.p, 8, cudaMemcpyDeviceToHost));
    if (P > postings_cap) fail(PLAID_INVALID_PARAMS, "postings capacity too small (need " + std::to_string(P) + ")");
    int end_bit = 32;
    while (end_bit < 64 && (K - 1) >> (end_bit - 32)) ++end_bit;
    size_t tmp_bytes = 0;
    PLAID_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_keys.p, d_sorted.p, P, 0, end_bit, st));
    Dev<uint8_t> d_tmp(tmp_bytes);
    PLAID_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp.p, tmp_bytes, d_keys.p, d_sorted.p, P, 0, end_bit, st));
    Dev<uint32_t> d_post(P);
    low_words_kernel<<<grid_cap(P, 256, 148 * 16), 256, 0, st>>>(d_sorted.p, P, d_post.p);
    PLAID_CUDA(cudaGetLastError());
    Dev<unsigned long long> d_offs(K + 1);
    size_t scan_bytes = 0;
    PLAID_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_counts.p, d_offs.p, K + 1, st));
    Dev<uint8_t> d_stmp(scan_bytes);
    PLAID_CUDA(cub::DeviceScan::ExclusiveSum(d_stmp.p, scan_bytes, d_counts.p, d_offs.p, K + 1, st));

    PLAID_CUDA(cudaMemcpy(codes, d_codes.p, T * 4, cudaMemcpyDeviceToHost));
    PLAID_CUDA(cudaMemcpy(residuals, d_res.p, T * bpt, cudaMemcpyDeviceToHost));
    PLAID_CUDA(cudaMemcpy(ivf_offsets, d_offs.p, (K + 1) * 8, cudaMemcpyDeviceToHost));
    PLAID_CUDA(cudaMemcpy(ivf_postings, d_post.p, P * 4, cudaMemcpyDeviceToHost));
    *num_postings = P;
}

// ---- index training: lir::build_index (indexer.cpp:197-282)
namespace {

// SplitMix64 (rng.hpp:11-56) for the sequential, seed-driven decisions.
struct HostRng {
    uint64_t s;
    explicit HostRng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return (double(next() >> 11) + 0.5) * 0x1.0p-53; }
    uint64_t below(uint64_t bound) { return bound ? next() % bound : 0; }
};
uint64_t mix_seed(uint64_t a, uint64_t b) { return HostRng(a ^ (0x9E3779B97F4A7C15ULL + (b << 6) + (b >> 2))).next(); }

// Seeded partial Fisher-Yates: `m` sorted picks from [0, n) (indexer.cpp:226-241, :95-106).
std::vector<uint64_t> partial_fisher_yates(uint64_t n, uint64_t m, uint64_t seed) {
    std::vector<uint64_t> all(n);
    for (uint64_t i = 0; i < n; ++i) all[i] = i;
    HostRng rng(seed);
    std::vector<uint64_t> picked(m);
    for (uint64_t i = 0; i < m; ++i) {
        const uint64_t j = i + rng.below(n - i);
        std::swap(all[i], all[j]);
        picked[i] = all[i];
    }
    std::sort(picked.begin(), picked.end());
    return picked;
}

float quantile_cutoff(const std::vector<float>& sorted, double q) {  // indexer.cpp:21-33
    const uint64_t n = sorted.size();
    const double pos = q * double(n);
    uint64_t rank = uint64_t(std::ceil(pos));
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    if (pos == std::floor(pos)) {
        const uint64_t lo = uint64_t(pos);
        if (lo >= 1 && lo < n) return 0.5f * (sorted[lo - 1] + sorted[lo]);
    }
    return sorted[rank - 1];
}

uint32_t bucket_for(const float* cut, uint32_t ncut, float x) {  // residual_codec.hpp:23-31
    uint32_t lo = 0, hi = ncut;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (cut[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// kmeans.cpp:36-74, on the host: it is a sequential scan with "stolen" state
bool repair_empty(const std::vector<float>& pts, uint64_t n, uint32_t dim, std::vector<float>& C, uint64_t k,
                  std::vector<uint32_t>& best, std::vector<float>& best_dot, std::vector<uint8_t>& stolen,
                  bool& changed) {
    std::vector<uint32_t> counts(k, 0);
    for (uint64_t j = 0; j < n; ++j) counts[best[j]]++;
    bool all_repaired = true;
    for (uint64_t c = 0; c < k; ++c) {
        if (counts[c] != 0) continue;
        uint64_t victim = n;
        float victim_dot = INFINITY;
        for (uint64_t j = 0; j < n; ++j) {
            if (stolen[j]) continue;
            if (counts[best[j]] <= 1) continue;
            if (best_dot[j] < victim_dot) {
                victim_dot = best_dot[j];
                victim = j;
            }
        }
        if (victim == n || victim_dot >= 1.0f - 1e-12f) {
            all_repaired = false;
            continue;
        }
        counts[best[victim]]--;
        std::copy_n(pts.data() + victim * dim, dim, C.data() + c * dim);
        best[victim] = uint32_t(c);
        best_dot[victim] = 1.0f;
        stolen[victim] = 1;
        counts[c] = 1;
        changed = true;
    }
    return all_repaired;
}

}  // namespace

// train_centroids (kmeans.cpp:78-175) with the heavy loops on the GPU: the
// seeding dots, every assignment pass (T x K in-order fp32 dots) and the mean
// sums; the seed-driven sequential choices (k-means++ picks, empty-cluster
// repair) on the host, in the reference's order — bit-identical centroids.
std::vector<float> train_centroids_gpu(const std::vector<float>& pts, uint64_t n, uint32_t dim, uint64_t k,
                                       uint64_t iters, uint64_t seed, int device) {
    if (k < 1) fail(PLAID_INVALID_PARAMS, "k must be >= 1");
    if (iters < 1) fail(PLAID_INVALID_PARAMS, "iters must be >= 1");
    if (n < k) fail(PLAID_TOO_FEW_POINTS, std::to_string(n) + " training points for k = " + std::to_string(k));
    DeviceGuard g(device);
    cudaStream_t st = nullptr;
    std::vector<float> C(k * dim);
    HostRng rng(seed);
    Dev<float> d_pts(n * dim), d_C(k * dim), d_bd(n), d_top(n);
    Dev<uint32_t> d_best(n);
    PLAID_CUDA(cudaMemcpy(d_pts.p, pts.data(), n * dim * 4, cudaMemcpyHostToDevice));
    const uint32_t sgrid = grid_cap(n, 256, 148 * 16);
    // k-means++ seeding: d^2 = 2 - 2 cos from the running best dot
    {
        const uint64_t first = rng.below(n);
        std::copy_n(pts.data() + first * dim, dim, C.data());
        PLAID_CUDA(cudaMemcpy(d_C.p, C.data(), dim * 4, cudaMemcpyHostToDevice));
        seed_update_kernel<<<sgrid, 256, dim * 4, st>>>(d_pts.p, n, dim, d_C.p, d_bd.p, 1);
        PLAID_CUDA(cudaGetLastError());
        std::vector<float> bd(n);
        for (uint64_t c = 1; c < k; ++c) {
            PLAID_CUDA(cudaMemcpy(bd.data(), d_bd.p, n * 4, cudaMemcpyDeviceToHost));
            double total = 0.0;
            for (uint64_t j = 0; j < n; ++j) total += std::max(0.0, 2.0 - 2.0 * double(bd[j]));
            uint64_t pick;
            if (total <= 0.0) {
                pick = rng.below(n);
            } else {
                const double r = rng.unit() * total;
                double cum = 0.0;
                pick = n - 1;
                for (uint64_t j = 0; j < n; ++j) {
                    cum += std::max(0.0, 2.0 - 2.0 * double(bd[j]));
                    if (cum > r) {
                        pick = j;
                        break;
                    }
                }
            }
            std::copy_n(pts.data() + pick * dim, dim, C.data() + c * dim);
            PLAID_CUDA(cudaMemcpy(d_C.p + c * dim, C.data() + c * dim, dim * 4, cudaMemcpyHostToDevice));
            seed_update_kernel<<<sgrid, 256, dim * 4, st>>>(d_pts.p, n, dim, d_C.p + c * dim, d_bd.p, 0);
            PLAID_CUDA(cudaGetLastError());
        }
    }
    const size_t smem = size_t(dim) * (kTokTile + kCentChunk) * sizeof(float);
    PLAID_CUDA(cudaFuncSetAttribute(assign_codes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    std::vector<uint32_t> best(n), members(n);
    std::vector<float> best_dot(n);
    std::vector<uint64_t> moff(k + 1);
    Dev<uint32_t> d_members(n);
    Dev<uint64_t> d_moff(k + 1);
    Dev<double> d_sums(k * dim);
    for (uint64_t it = 0; it <= iters; ++it) {
        PLAID_CUDA(cudaMemcpy(d_C.p, C.data(), k * dim * 4, cudaMemcpyHostToDevice));
        assign_codes_kernel<<<uint32_t((n + kTokTile - 1) / kTokTile), kTokTile, smem, st>>>(
            d_pts.p, n, d_C.p, uint32_t(k), dim, d_best.p, d_top.p);
        PLAID_CUDA(cudaGetLastError());
        PLAID_CUDA(cudaMemcpy(best.data(), d_best.p, n * 4, cudaMemcpyDeviceToHost));
        PLAID_CUDA(cudaMemcpy(best_dot.data(), d_top.p, n * 4, cudaMemcpyDeviceToHost));
        std::vector<uint8_t> stolen(n, 0);
        bool changed = false;
        for (int round = 0; round < 16; ++round)
            if (repair_empty(pts, n, dim, C, k, best, best_dot, stolen, changed)) break;
        if (it == iters) break;  // final pass fixes assignments/empties only
        // members of each cluster in point order (stable counting sort)
        std::fill(moff.begin(), moff.end(), 0);
        for (uint64_t j = 0; j < n; ++j) moff[best[j] + 1]++;
        for (uint64_t c = 0; c < k; ++c) moff[c + 1] += moff[c];
        {
            std::vector<uint64_t> cur(moff.begin(), moff.end() - 1);
            for (uint64_t j = 0; j < n; ++j) members[cur[best[j]]++] = uint32_t(j);
        }
        if (changed) PLAID_CUDA(cudaMemcpy(d_C.p, C.data(), k * dim * 4, cudaMemcpyHostToDevice));
        PLAID_CUDA(cudaMemcpy(d_members.p, members.data(), n * 4, cudaMemcpyHostToDevice));
        PLAID_CUDA(cudaMemcpy(d_moff.p, moff.data(), (k + 1) * 8, cudaMemcpyHostToDevice));
        mean_sum_kernel<<<uint32_t((k * dim + 255) / 256), 256, 0, st>>>(d_pts.p, dim, d_members.p, d_moff.p, k,
                                                                        d_sums.p);
        mean_norm_kernel<<<uint32_t((k + 127) / 128), 128, 0, st>>>(d_sums.p, d_moff.p, k, dim, d_C.p);
        PLAID_CUDA(cudaGetLastError());
        PLAID_CUDA(cudaMemcpy(C.data(), d_C.p, k * dim * 4, cudaMemcpyDeviceToHost));
    }
    return C;
}

// lir::build_index (indexer.cpp:197-282): sample, train_centroids,
// assign_codes, train_quantizer (indexer.cpp:74-147), residuals, IVF.
void build_index_host(const float* emb, const uint32_t* doclens, uint64_t N, uint32_t dim, uint32_t nbits, uint64_t K,
                      uint64_t iters, uint64_t seed, int device, float* centroids_out, float* cutoffs_out,
                      float* weights_out, uint64_t* k_out, uint32_t* codes, uint8_t* residuals, uint64_t* ivf_offsets,
                      uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings) {
    uint64_t T = 0;
    for (uint64_t p = 0; p < N; ++p) T += doclens[p];
    if (N == 0 || T == 0) fail(PLAID_EMPTY_CORPUS, "cannot index an empty corpus");
    if (nbits != 1 && nbits != 2 && nbits != 4) fail(PLAID_PACKING_UNSUPPORTED, "nbits must be one of {1,2,4}");
    if (dim == 0 || dim % (8 / nbits) != 0)
        fail(PLAID_PACKING_UNSUPPORTED, "dim " + std::to_string(dim) + " not divisible by " +
                                            std::to_string(8 / nbits) + " for nbits " + std::to_string(nbits));
    if (N > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "corpora above 2^32 passages are not supported");
    validate_query_host(emb, T, dim, dim);  // CorpusEmbeddings::create's unit rows (types.cpp:10-19)
    uint64_t k = K;
    if (!k) {  // auto_num_centroids (indexer.cpp:37-43)
        const uint64_t e = uint64_t(std::ceil(std::log2(double(T)) / 2.0));
        k = std::min<uint64_t>(std::max<uint64_t>(uint64_t(1) << e, 1), T);
    }
    if (k > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "centroid count must be in [1, 2^32)");
    // training sample: uniform over tokens, >= K rows, capped at 2^20
    const double fraction = std::min(1.0, double(uint64_t(1) << 20) / double(T));
    uint64_t sample_size = uint64_t(std::ceil(fraction * double(T)));
    sample_size = std::clamp<uint64_t>(sample_size, std::min(T, k), T);
    std::vector<float> sample;
    if (sample_size < T) {
        const std::vector<uint64_t> picked = partial_fisher_yates(T, sample_size, mix_seed(seed, 0x5A75A75A75A75A75ULL));
        sample.resize(sample_size * dim);
        for (uint64_t i = 0; i < sample_size; ++i) std::copy_n(emb + picked[i] * dim, dim, sample.data() + i * dim);
    } else {
        sample.assign(emb, emb + T * dim);
    }
    const std::vector<float> C = train_centroids_gpu(sample, sample_size, dim, k, iters, seed, device);
    // codes of every token (the encode pass), then the quantizer, then residuals + IVF
    DeviceGuard g(device);
    Dev<float> d_emb(T * dim), d_C(k * dim);
    Dev<uint32_t> d_codes(T);
    PLAID_CUDA(cudaMemcpy(d_emb.p, emb, T * dim * 4, cudaMemcpyHostToDevice));
    PLAID_CUDA(cudaMemcpy(d_C.p, C.data(), k * dim * 4, cudaMemcpyHostToDevice));
    const size_t smem = size_t(dim) * (kTokTile + kCentChunk) * sizeof(float);
    PLAID_CUDA(cudaFuncSetAttribute(assign_codes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    assign_codes_kernel<<<uint32_t((T + kTokTile - 1) / kTokTile), kTokTile, smem>>>(d_emb.p, T, d_C.p, uint32_t(k),
                                                                                     dim, d_codes.p, nullptr);
    PLAID_CUDA(cudaGetLastError());
    std::vector<uint32_t> all_codes(T);
    PLAID_CUDA(cudaMemcpy(all_codes.data(), d_codes.p, T * 4, cudaMemcpyDeviceToHost));
    // train_quantizer (indexer.cpp:74-147): residual components of a token
    // subset, quantile cutoffs, bucket means (sequential double sums)
    const uint64_t max_tokens = std::max<uint64_t>(1, (uint64_t(1) << 20) / std::max<uint64_t>(dim, 1));
    std::vector<uint64_t> tok;
    if (T <= max_tokens) {
        tok.resize(T);
        for (uint64_t i = 0; i < T; ++i) tok[i] = i;
    } else {
        tok = partial_fisher_yates(T, max_tokens, mix_seed(seed, 0x71D67FFFEDA60000ULL));
    }
    std::vector<float> pool(tok.size() * dim);
    for (uint64_t i = 0; i < tok.size(); ++i) {
        const float* v = emb + tok[i] * dim;
        const float* c = C.data() + uint64_t(all_codes[tok[i]]) * dim;
        for (uint32_t d = 0; d < dim; ++d) pool[i * dim + d] = v[d] - c[d];
    }
    std::vector<float> sorted = pool;
    std::sort(sorted.begin(), sorted.end());
    const uint32_t nb = 1u << nbits;
    float cut[16] = {}, w[16] = {};
    for (uint32_t i = 1; i < nb; ++i) cut[i - 1] = quantile_cutoff(sorted, double(i) / double(nb));
    double sums[16] = {};
    uint64_t counts[16] = {};
    for (float x : pool) {
        const uint32_t b = bucket_for(cut, nb - 1, x);
        sums[b] += x;
        counts[b]++;
    }
    for (uint32_t b = 0; b < nb; ++b)
        w[b] = counts[b] > 0 ? float(sums[b] / double(counts[b])) : (b == 0 ? cut[0] : cut[b - 1]);
    // residuals + IVF: the encode pass with the trained centroids and cutoffs
    plaid_encode_desc ed{};
    ed.dim = dim;
    ed.nbits = nbits;
    ed.num_centroids = k;
    ed.num_passages = N;
    ed.num_embeddings = T;
    ed.embeddings = emb;
    ed.doclens = doclens;
    ed.centroids = C.data();
    ed.bucket_cutoffs = cut;
    encode_host(ed, device, codes, residuals, ivf_offsets, ivf_postings, postings_cap, num_postings);
    std::memcpy(centroids_out, C.data(), k * dim * 4);
    std::memcpy(cutoffs_out, cut, (nb - 1) * 4);
    std::memcpy(weights_out, w, nb * 4);
    *k_out = k;
}

}  // namespace plaid
