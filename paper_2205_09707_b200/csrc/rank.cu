// rank.cu — stage 4, residual decompression fused with exact MaxSim
// (pipeline.cpp:165-225, residual_codec.cpp:97-132, maxsim.cpp:66-104).
//
// One CTA (4 warps) per finalist passage; tokens are processed in tiles of 32:
//   1. decompress: each warp unpacks its tokens' b-bit fields straight from the
//      packed bytes (LSB-first, table[v][j] = (v >> b*j) & (2^b-1),
//      residual_codec.cpp:42-59) and adds the bucket weight to the centroid
//      row: v = C[code] + w[idx] (fp32, 128-bit loads of C);
//   2. normalise: ||v||^2 in fp64, in order over d, inv = float(1/sqrt) —
//      exactly residual_codec.cpp:124-129;
//   3. MaxSim: lane = token, warp w scores query tokens [8w, 8w+8) with
//      in-order fp32 dots (maxsim.cpp:89-99), then a per-query max across the
//      tile; the running max lives in shared memory across tiles;
//   4. the score is the in-order fp32 sum over query tokens.
// The decompressed rows never leave shared memory (the reference materialises
// a T4 x d fp32 buffer; here the only HBM traffic is codes, packed residuals
// and centroid rows).  Output: one 64-bit (score, pid) key per passage.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr uint32_t kThreads = 128;
constexpr uint32_t kTile = 32;

struct Weights {
    float w[16];
};

// Decompress token `tok` into v (dim floats) cooperatively across a warp.
__device__ __forceinline__ void decompress_token(const float* __restrict__ C, uint32_t dim,
                                                 uint32_t nbits, const Weights& W, uint32_t code,
                                                 const uint8_t* __restrict__ bytes, float* v) {
    const uint32_t lane = dev::lane_id();
    const uint32_t per = 8 / nbits, mask = (1u << nbits) - 1;
    const float4* crow = reinterpret_cast<const float4*>(C + uint64_t(code) * dim);
    for (uint32_t d4 = lane; d4 < dim / 4; d4 += 32) {
        const float4 c = __ldg(crow + d4);
        const uint32_t d = d4 * 4;
        float r[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t dd = d + e;
            const uint32_t idx = (uint32_t(__ldg(bytes + dd / per)) >> (nbits * (dd % per))) & mask;
            r[e] = W.w[idx];
        }
        float4 o;
        o.x = __fadd_rn(c.x, r[0]);
        o.y = __fadd_rn(c.y, r[1]);
        o.z = __fadd_rn(c.z, r[2]);
        o.w = __fadd_rn(c.w, r[3]);
        reinterpret_cast<float4*>(v)[d4] = o;
    }
}

// In-order fp64 norm (residual_codec.cpp:124-129) -> scale factor (1.0f if 0).
__device__ __forceinline__ float inv_norm(const float* v, uint32_t dim) {
    double acc = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
        const double x = double(v[d]);
        acc = __dadd_rn(acc, __dmul_rn(x, x));
    }
    return acc > 0.0 ? float(1.0 / sqrt(acc)) : 1.0f;
}

__global__ void __launch_bounds__(kThreads)
rank_exact_kernel(const float* __restrict__ C, const uint32_t* __restrict__ codes,
                  const uint8_t* __restrict__ residuals, const uint32_t* __restrict__ doclens,
                  const uint64_t* __restrict__ offsets, uint32_t dim, uint32_t nbits, Weights W,
                  const float* __restrict__ Q, uint32_t rows, const uint32_t* __restrict__ ids,
                  const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                  uint64_t* __restrict__ out_keys) {
    dev::pdl_wait();
    extern __shared__ __align__(16) float sm[];
    const uint32_t pitch = dim + 4;
    float* q_s = sm;                    // 32 x pitch
    float* v_s = sm + 32 * pitch;       // kTile x pitch
    __shared__ float inv_s[kTile];
    __shared__ float run_s[32];
    const uint32_t lane = dev::lane_id(), warp = threadIdx.x >> 5;
    const uint64_t bpt = uint64_t(nbits) * dim / 8;

    for (uint32_t idx = threadIdx.x; idx < 32 * dim; idx += kThreads) {
        const uint32_t i = idx / dim, d = idx % dim;
        q_s[i * pitch + d] = i < rows ? Q[i * dim + d] : 0.0f;
    }
    const uint64_t n = *d_n;
    for (uint64_t p = blockIdx.x; p < n; p += gridDim.x) {
        const uint32_t pid = ids ? ids[p] : dev::key_id(keys[p]);
        const uint64_t off = offsets[pid];
        const uint32_t len = doclens[pid];
        if (threadIdx.x < 32) run_s[threadIdx.x] = -INFINITY;
        for (uint32_t t0 = 0; t0 < len; t0 += kTile) {
            const uint32_t nt = len - t0 < kTile ? len - t0 : kTile;
            __syncthreads();  // previous tile's v_s fully consumed
            for (uint32_t tt = warp; tt < nt; tt += kThreads / 32) {
                const uint64_t tok = off + t0 + tt;
                decompress_token(C, dim, nbits, W, __ldg(codes + tok), residuals + tok * bpt,
                                 v_s + tt * pitch);
            }
            __syncthreads();
            if (threadIdx.x < nt) inv_s[threadIdx.x] = inv_norm(v_s + threadIdx.x * pitch, dim);
            __syncthreads();
            for (uint32_t e = threadIdx.x; e < nt * dim; e += kThreads) {
                const uint32_t tt = e / dim, d = e % dim;
                v_s[tt * pitch + d] = __fmul_rn(v_s[tt * pitch + d], inv_s[tt]);
            }
            __syncthreads();
            // MaxSim: lane = token, warp w -> query tokens 8w .. 8w+7
            const uint32_t i0 = warp * 8;
            if (i0 < rows) {
                float a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = 0.0f;
                const float4* vr = reinterpret_cast<const float4*>(v_s + (lane < nt ? lane : 0) * pitch);
                for (uint32_t d4 = 0; d4 < dim / 4; ++d4) {
                    const float4 v = vr[d4];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float4 q = reinterpret_cast<const float4*>(q_s + (i0 + u) * pitch)[d4];
                        float x = a[u];
                        x = dev::madd_rn(x, q.x, v.x);
                        x = dev::madd_rn(x, q.y, v.y);
                        x = dev::madd_rn(x, q.z, v.z);
                        x = dev::madd_rn(x, q.w, v.w);
                        a[u] = x;
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float m = dev::warp_max(lane < nt ? a[u] : -INFINITY);
                    if (lane == uint32_t(u) && i0 + u < rows) run_s[i0 + u] = dev::max_gt(run_s[i0 + u], m);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float total = 0.0f;
            for (uint32_t i = 0; i < rows; ++i) total = __fadd_rn(total, run_s[i]);
            out_keys[p] = dev::make_key(total, pid);
        }
        __syncthreads();
    }
}

// ---- d = 128 fast path ---------------------------------------------------------
// One warp per finalist passage, lane = QUERY token: each lane keeps its
// query row q_i (128 fp32) in registers for the whole kernel, so the
// per-passage max over tokens is thread-local and no lane idles on short
// passages.  Per chunk of <= 32 passage tokens:
//   1. decompress (lane = 4 dims, coalesced 512-byte centroid rows, the
//      lane's 4 bucket indices from one residual byte at b=2) into the warp's
//      shared-memory tile v[t][d] (pitch 132: conflict-free for both the
//      row-per-lane and the broadcast access below);
//   2. lane = token: in-order fp64 norm of its row and in-place scaling
//      (residual_codec.cpp:124-129);
//   3. lane = query: for each token, the in-order fp32 dot q_i . v_t with v_t
//      broadcast from shared memory (LDS.128), two tokens interleaved so two
//      dependent add chains are in flight; run_i = max(run_i, dot).
// Then score = in-order fp32 sum of run_i over i (maxsim.cpp:89-99).
constexpr uint32_t kR128Warps = 4;
constexpr uint32_t kR128Pitch = 132;
constexpr uint32_t kR128Chunk = 32;

template <int NB>
__global__ void __launch_bounds__(kR128Warps * 32, 3)
rank128_kernel(const float* __restrict__ C, const uint32_t* __restrict__ codes,
               const uint8_t* __restrict__ residuals, const uint32_t* __restrict__ doclens,
               const uint64_t* __restrict__ offsets, Weights W, const float* __restrict__ Q, uint32_t rows,
               const uint32_t* __restrict__ ids, const uint64_t* __restrict__ keys,
               const uint64_t* __restrict__ d_n, uint64_t* __restrict__ out_keys) {
    dev::pdl_wait();
    extern __shared__ __align__(16) float sm[];
    __shared__ float w_s[16];
    constexpr uint32_t kBpt = NB * 128 / 8;  // residual bytes per token
    const uint32_t lane = dev::lane_id(), warp = threadIdx.x >> 5;
    float* v_s = sm + warp * kR128Chunk * kR128Pitch;
    if (threadIdx.x < 16) w_s[threadIdx.x] = W.w[threadIdx.x];
    __syncthreads();

    float q[128];
    {
        const float4* qr = reinterpret_cast<const float4*>(Q + uint64_t(lane < rows ? lane : 0) * 128);
#pragma unroll
        for (int d4 = 0; d4 < 32; ++d4) {
            const float4 x = lane < rows ? __ldg(qr + d4) : make_float4(0.f, 0.f, 0.f, 0.f);
            q[4 * d4] = x.x, q[4 * d4 + 1] = x.y, q[4 * d4 + 2] = x.z, q[4 * d4 + 3] = x.w;
        }
    }
    const uint64_t n = *d_n;
    const uint64_t nwarps = uint64_t(gridDim.x) * kR128Warps;
    // passage p -> CTA p % grid: consecutive finalists land on different SMs
    for (uint64_t p = uint64_t(warp) * gridDim.x + blockIdx.x; p < n; p += nwarps) {
        const uint32_t pid = ids ? ids[p] : dev::key_id(keys[p]);
        const uint64_t off = offsets[pid];
        const uint32_t len = doclens[pid];
        float run = -INFINITY;
        for (uint32_t t0 = 0; t0 < len; t0 += kR128Chunk) {
            const uint32_t nt = len - t0 < kR128Chunk ? len - t0 : kR128Chunk;
            const uint32_t code_l = lane < nt ? __ldg(codes + off + t0 + lane) : 0u;
            // 1. decompress: v = C[code] + w[idx], lane = dims 4*lane .. 4*lane+3
#pragma unroll 8
            for (uint32_t tt = 0; tt < nt; ++tt) {
                const uint32_t code = __shfl_sync(0xffffffffu, code_l, tt);
                const float4 c = __ldg(reinterpret_cast<const float4*>(C + uint64_t(code) * 128) + lane);
                const uint8_t* rb = residuals + (off + t0 + tt) * kBpt;
                uint32_t bits, sh;
                if (NB == 1) {
                    bits = __ldg(rb + (lane >> 1));
                    sh = (lane & 1) * 4;
                } else if (NB == 2) {
                    bits = __ldg(rb + lane);
                    sh = 0;
                } else {
                    bits = __ldg(reinterpret_cast<const uint16_t*>(rb) + lane);
                    sh = 0;
                }
                constexpr uint32_t mask = (1u << NB) - 1;
                float4 v;
                v.x = __fadd_rn(c.x, w_s[(bits >> (sh + 0 * NB)) & mask]);
                v.y = __fadd_rn(c.y, w_s[(bits >> (sh + 1 * NB)) & mask]);
                v.z = __fadd_rn(c.z, w_s[(bits >> (sh + 2 * NB)) & mask]);
                v.w = __fadd_rn(c.w, w_s[(bits >> (sh + 3 * NB)) & mask]);
                reinterpret_cast<float4*>(v_s + tt * kR128Pitch)[lane] = v;
            }
            __syncwarp();
            // 2. lane = token: in-order fp64 norm, then v *= inv
            if (lane < nt) {
                float4* row = reinterpret_cast<float4*>(v_s + lane * kR128Pitch);
                double acc = 0.0;
#pragma unroll 8
                for (int d4 = 0; d4 < 32; ++d4) {
                    const float4 x = row[d4];
                    acc = __dadd_rn(acc, __dmul_rn(double(x.x), double(x.x)));
                    acc = __dadd_rn(acc, __dmul_rn(double(x.y), double(x.y)));
                    acc = __dadd_rn(acc, __dmul_rn(double(x.z), double(x.z)));
                    acc = __dadd_rn(acc, __dmul_rn(double(x.w), double(x.w)));
                }
                if (acc > 0.0) {
                    const float inv = float(1.0 / sqrt(acc));
#pragma unroll 8
                    for (int d4 = 0; d4 < 32; ++d4) {
                        float4 x = row[d4];
                        x.x = __fmul_rn(x.x, inv), x.y = __fmul_rn(x.y, inv);
                        x.z = __fmul_rn(x.z, inv), x.w = __fmul_rn(x.w, inv);
                        row[d4] = x;
                    }
                }
            }
            __syncwarp();
            // 3. lane = query: in-order dots against broadcast token rows
            for (uint32_t tt = 0; tt < nt; tt += 2) {
                const uint32_t t1 = tt + 1 < nt ? tt + 1 : tt;
                const float4* r0 = reinterpret_cast<const float4*>(v_s + tt * kR128Pitch);
                const float4* r1 = reinterpret_cast<const float4*>(v_s + t1 * kR128Pitch);
                float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
                for (int d4 = 0; d4 < 32; ++d4) {
                    const float4 a = r0[d4], b = r1[d4];
                    s0 = dev::madd_rn(s0, q[4 * d4 + 0], a.x);
                    s1 = dev::madd_rn(s1, q[4 * d4 + 0], b.x);
                    s0 = dev::madd_rn(s0, q[4 * d4 + 1], a.y);
                    s1 = dev::madd_rn(s1, q[4 * d4 + 1], b.y);
                    s0 = dev::madd_rn(s0, q[4 * d4 + 2], a.z);
                    s1 = dev::madd_rn(s1, q[4 * d4 + 2], b.z);
                    s0 = dev::madd_rn(s0, q[4 * d4 + 3], a.w);
                    s1 = dev::madd_rn(s1, q[4 * d4 + 3], b.w);
                }
                run = dev::max_gt(run, s0);
                run = dev::max_gt(run, s1);  // t1 == tt on an odd tail: same value
            }
            __syncwarp();
        }
        // in-order sum over query tokens
        float total = 0.0f;
        for (uint32_t i = 0; i < rows; ++i) total = __fadd_rn(total, __shfl_sync(0xffffffffu, run, i));
        if (lane == 0) out_keys[p] = dev::make_key(total, pid);
    }
}

// ---- per-stage entry points -------------------------------------------------

__global__ void unpack_kernel(const uint8_t* __restrict__ packed, uint64_t n, uint32_t nbits,
                              uint8_t* __restrict__ out) {
    dev::pdl_wait();
    const uint32_t per = 8 / nbits, mask = (1u << nbits) - 1;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = packed[i];
        for (uint32_t j = 0; j < per; ++j) out[i * per + j] = uint8_t((v >> (nbits * j)) & mask);
    }
}

// One warp per token: v = normalize(C[code] + w[idx]) (residual_codec.cpp:97-132).
__global__ void reconstruct_kernel(const float* __restrict__ C, uint32_t dim, uint32_t nbits, Weights W,
                                   const uint32_t* __restrict__ codes, uint64_t n,
                                   const uint8_t* __restrict__ residuals, float* __restrict__ out) {
    dev::pdl_wait();
    const uint64_t bpt = uint64_t(nbits) * dim / 8;
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); t < n; t += nw) {
        float* v = out + t * dim;
        decompress_token(C, dim, nbits, W, codes[t], residuals + t * bpt, v);
        __syncwarp();
        float inv = 0.0f;
        if (dev::lane_id() == 0) inv = inv_norm(v, dim);
        inv = __shfl_sync(0xffffffffu, inv, 0);
        for (uint32_t d = dev::lane_id(); d < dim; d += 32) v[d] = __fmul_rn(v[d], inv);
        __syncwarp();
    }
}

// maxsim.cpp:31-64: one warp per passage, lane = query column (nq <= 32).
__global__ void maxsim_packed_kernel(const float* __restrict__ scores, uint32_t nq,
                                     const uint64_t* __restrict__ offsets, uint64_t np,
                                     float* __restrict__ out) {
    dev::pdl_wait();
    const uint32_t lane = dev::lane_id();
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); p < np; p += nw) {
        float acc = -INFINITY;
        for (uint64_t t = offsets[p]; t < offsets[p + 1]; ++t)
            if (lane < nq) acc = dev::max_gt(acc, scores[t * nq + lane]);
        float total = 0.0f;
        for (uint32_t j = 0; j < nq; ++j) total = __fadd_rn(total, __shfl_sync(0xffffffffu, acc, j));
        if (lane == 0) out[p] = total;
    }
}

// maxsim.cpp:66-104: one warp per passage, lane = query token, in-order dots.
__global__ void maxsim_embeddings_kernel(const float* __restrict__ Q, uint32_t rows, uint32_t dim,
                                         const float* __restrict__ emb,
                                         const uint64_t* __restrict__ offsets, uint64_t np,
                                         float* __restrict__ out) {
    dev::pdl_wait();
    const uint32_t lane = dev::lane_id();
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const float* q = Q + uint64_t(lane < rows ? lane : 0) * dim;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); p < np; p += nw) {
        float acc = -INFINITY;
        for (uint64_t t = offsets[p]; t < offsets[p + 1]; ++t) {
            const float* v = emb + t * dim;
            float s = 0.0f;
            for (uint32_t d = 0; d < dim; ++d) s = dev::madd_rn(s, q[d], v[d]);
            acc = dev::max_gt(acc, s);
        }
        float total = 0.0f;
        for (uint32_t j = 0; j < rows; ++j) total = __fadd_rn(total, __shfl_sync(0xffffffffu, acc, j));
        if (lane == 0) out[p] = total;
    }
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

}  // namespace

namespace launch {

void rank_exact(const IndexView& ix, const float* d_q, uint32_t rows, const uint32_t* d_ids,
                const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t* d_out_keys,
                const RankScratch* scratch, cudaStream_t st) {
    if (nmax == 0) return;
    Weights W;
    for (int i = 0; i < 16; ++i) W.w[i] = ix.weights[i];
    if (ix.dim == 128 && rows <= 32 && scratch && rank_stream128(ix, d_q, rows, d_ids, d_keys, d_n, nmax, d_out_keys, *scratch, st))
        return;
    if (ix.dim == 128 && rows <= 32) {
        const size_t smem = size_t(kR128Warps) * kR128Chunk * kR128Pitch * sizeof(float);
        static launch::PerDeviceOnce cfg128;
        if (cfg128.first()) {
            cudaFuncSetAttribute(rank128_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            cudaFuncSetAttribute(rank128_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            cudaFuncSetAttribute(rank128_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        }
        // 3 CTAs (12 warps) per SM, one warp per finalist
        uint64_t blocks = uint64_t(sm_count()) * 3;
        if (blocks > nmax) blocks = nmax;
        auto k = ix.nbits == 1 ? rank128_kernel<1> : ix.nbits == 2 ? rank128_kernel<2> : rank128_kernel<4>;
        ::plaid::launch::pdl(k, uint32_t(blocks), kR128Warps * 32, smem, st, ix.centroids, ix.codes, ix.residuals, ix.doclens,
                                                           ix.offsets, W, d_q, rows, d_ids, d_keys, d_n,
                                                           d_out_keys);
        count_launch();
        return;
    }
    const size_t smem = size_t(32 + kTile) * (ix.dim + 4) * sizeof(float);
    static launch::PerDeviceOnce configured;
    if (configured.first()) {
        cudaFuncSetAttribute(rank_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    uint64_t blocks = nmax;
    const uint64_t cap = uint64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    ::plaid::launch::pdl(rank_exact_kernel, uint32_t(blocks), kThreads, smem, st, 
        ix.centroids, ix.codes, ix.residuals, ix.doclens, ix.offsets, ix.dim, ix.nbits, W, d_q, rows,
        d_ids, d_keys, d_n, d_out_keys);
    count_launch();
}

void unpack_via_lut(const uint8_t* d_packed, uint64_t n, uint32_t nbits, uint8_t* d_out,
                    cudaStream_t st) {
    if (!n) return;
    uint64_t b = (n + 255) / 256;
    ::plaid::launch::pdl(unpack_kernel, uint32_t(b > 4096 ? 4096 : b), 256, 0, st, d_packed, n, nbits, d_out);
    count_launch();
}

void reconstruct(const IndexView& ix, const uint32_t* d_codes, uint64_t n, const uint8_t* d_residuals,
                 float* d_out, cudaStream_t st) {
    if (!n) return;
    Weights W;
    for (int i = 0; i < 16; ++i) W.w[i] = ix.weights[i];
    uint64_t b = (n + 7) / 8;
    ::plaid::launch::pdl(reconstruct_kernel, uint32_t(b > 4096 ? 4096 : b), 256, 0, st, ix.centroids, ix.dim, ix.nbits, W,
                                                                      d_codes, n, d_residuals, d_out);
    count_launch();
}

void maxsim_packed(const float* d_scores, uint32_t nq, const uint64_t* d_offsets, uint64_t np,
                   float* d_out, cudaStream_t st) {
    if (!np) return;
    uint64_t b = (np + 7) / 8;
    ::plaid::launch::pdl(maxsim_packed_kernel, uint32_t(b > 4096 ? 4096 : b), 256, 0, st, d_scores, nq, d_offsets, np, d_out);
    count_launch();
}

void maxsim_embeddings(const float* d_q, uint32_t rows, uint32_t dim, const float* d_emb,
                       const uint64_t* d_offsets, uint64_t np, float* d_out, cudaStream_t st) {
    if (!np) return;
    uint64_t b = (np + 7) / 8;
    ::plaid::launch::pdl(maxsim_embeddings_kernel, uint32_t(b > 4096 ? 4096 : b), 256, 0, st, d_q, rows, dim, d_emb,
                                                                            d_offsets, np, d_out);
    count_launch();
}

}  // namespace launch
}  // namespace plaid
