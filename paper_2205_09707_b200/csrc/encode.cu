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
// k-means and the quantizer fit (kmeans.cpp, indexer.cpp:74-147) stay on the
// host reference: they are order-sensitive sequential reductions that only
// see a <= 2^20-row sample.
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
                    uint32_t* __restrict__ codes) {
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
    if (t0 + tid < T) codes[t0 + tid] = arg;
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
                                                                                        dim, d_codes.p);
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

}  // namespace plaid
