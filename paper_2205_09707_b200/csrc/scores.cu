// scores.cu — stage 1 on CUDA cores, bit-exact with the reference:
//   S[c][i] = dot(C[c], Q[i]) in order over d, mul-then-add (pipeline.cpp:26-50,
//   types.hpp:18-22), row max (pipeline.cpp:40-46), keep bit (max >= t_cs,
//   pipeline.cpp:89-95) and the per-token top-nprobe centroid keys
//   (score desc, id asc; pipeline.cpp:65-73) fused into the same pass.
//
// Layout: C is K x dim row-major in HBM; S is K x 32 (row pitch 128 B) so the
// stage-2/3 row gathers are one 128-byte line per centroid.
//
// Work split: each warp owns chunks of 32 consecutive centroids (one keep-bit
// word) and walks them in groups of G=16; lane i is query token i.  The group's
// 16 C rows are staged in shared memory and read as broadcast LDS.128; the
// query rows sit in shared memory with a +4 float pad so the per-lane LDS.128
// is conflict-free.  Per 4 dims a lane issues 1 + 16 LDS.128 for 128 fp32 ops.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "device.cuh"
#include "fused.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr int kG = 16;           // centroids per group
constexpr int kWarpsPerBlock = 8;
constexpr int kBlocksPerSm = 2;

template <int NP>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kBlocksPerSm)
scores_exact_kernel(const float* __restrict__ C, uint64_t K, uint32_t dim,
                    const float* __restrict__ Q, uint32_t rows, float t_cs,
                    float* __restrict__ S, float* __restrict__ rowmax,
                    uint32_t* __restrict__ keep_bits, uint64_t* __restrict__ partial) {
    dev::pdl_wait();
    extern __shared__ __align__(16) float smem[];
    const uint32_t qpitch = dim + 4;
    float* q_s = smem;                                   // 32 x (dim+4)
    float* c_all = smem + 32 * qpitch;                   // warps x G x dim
    const uint32_t lane = dev::lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    float* c_s = c_all + warp * kG * dim;

    for (uint32_t idx = threadIdx.x; idx < 32 * dim; idx += blockDim.x) {
        uint32_t i = idx / dim, d = idx % dim;
        q_s[i * qpitch + d] = i < rows ? Q[i * dim + d] : 0.0f;
    }
    __syncthreads();

    uint64_t top[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) top[j] = 0;  // below every real key

    const uint64_t nchunks = (K + 31) / 32;
    const uint64_t gwarp = uint64_t(blockIdx.x) * kWarpsPerBlock + warp;
    const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerBlock;
    const float4* qrow = reinterpret_cast<const float4*>(q_s + lane * qpitch);

    for (uint64_t chunk = gwarp; chunk < nchunks; chunk += nwarps) {
        uint32_t keep_word = 0;
        for (int g = 0; g < 32 / kG; ++g) {
            const uint64_t c0 = chunk * 32 + g * kG;
            // centroids of this group (0 past the end of a partial last chunk)
            const uint32_t nc = c0 >= K ? 0u : uint32_t(K - c0 < kG ? K - c0 : kG);
            // stage the group's rows (contiguous in HBM) into shared memory
            const float4* src = reinterpret_cast<const float4*>(C + c0 * dim);
            float4* dst = reinterpret_cast<float4*>(c_s);
            const uint32_t n4 = nc * dim / 4, tot4 = kG * dim / 4;
            __syncwarp();
            for (uint32_t v = lane; v < tot4; v += 32)
                dst[v] = v < n4 ? __ldcs(src + v) : make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();

            float acc[kG];
#pragma unroll
            for (int c = 0; c < kG; ++c) acc[c] = 0.0f;
            const float4* crow = reinterpret_cast<const float4*>(c_s);
            const uint32_t dim4 = dim / 4;
            for (uint32_t d4 = 0; d4 < dim4; ++d4) {
                const float4 q = qrow[d4];
#pragma unroll
                for (int c = 0; c < kG; ++c) {
                    const float4 cv = crow[c * dim4 + d4];
                    float a = acc[c];
                    a = dev::madd_rn(a, cv.x, q.x);
                    a = dev::madd_rn(a, cv.y, q.y);
                    a = dev::madd_rn(a, cv.z, q.z);
                    a = dev::madd_rn(a, cv.w, q.w);
                    acc[c] = a;
                }
            }
            float my_max = -INFINITY;
#pragma unroll
            for (int c = 0; c < kG; ++c) {
                if (c < int(nc)) {
                    S[(c0 + c) * kScoresPitch + lane] = acc[c];
                    float m = dev::warp_max(lane < rows ? acc[c] : -INFINITY);
                    if (lane == uint32_t(c)) my_max = m;
                    if (m >= t_cs) keep_word |= 1u << (g * kG + c);
                    if (lane < rows) dev::topn_insert<NP>(top, dev::make_key(acc[c], uint32_t(c0 + c)));
                }
            }
            if (lane < nc) rowmax[c0 + lane] = my_max;
        }
        if (lane == 0) keep_bits[chunk] = keep_word;
    }
    uint64_t* out = partial + (gwarp * 32 + lane) * NP;
#pragma unroll
    for (int j = 0; j < NP; ++j) out[j] = top[j];
}

// One CTA: token i's best NP keys over the nwarps partial lists, left
// descending in lists[0..NP) (lists: blockDim x NP u64 of shared memory).
// Latency-shaped: each thread has all of its lists' loads in flight at once
// (the 8 epilogue warps of every S_cq CTA leave ~1200 lists per token), then
// a butterfly of shuffles merges the warp's lists (the sets are disjoint at
// every level, so the unique-key insert applies) and warp 0 merges the warps.
template <int NP>
__device__ void merge_token_lists(const uint64_t* __restrict__ partial, uint32_t nwarps, uint32_t i,
                                  uint64_t* lists) {
    if constexpr (NP > 8) {  // long lists: tree of two-pointer merges
        uint64_t top[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) top[j] = 0;
        for (uint32_t w = threadIdx.x; w < nwarps; w += blockDim.x) {
            const uint64_t* l = partial + (uint64_t(w) * 32 + i) * NP;
#pragma unroll
            for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, l[j]);
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) lists[threadIdx.x * NP + j] = top[j];
        __syncthreads();
        for (uint32_t s = blockDim.x / 2; s > 0; s >>= 1) {
            const bool active = threadIdx.x < s;
            uint64_t out[NP];
            if (active) {  // two-pointer merge of two descending lists, keep NP
                const uint64_t* a = lists + threadIdx.x * NP;
                const uint64_t* b = lists + (threadIdx.x + s) * NP;
                int ia = 0, ib = 0;
#pragma unroll
                for (int j = 0; j < NP; ++j) {
                    uint64_t va = ia < NP ? a[ia] : 0, vb = ib < NP ? b[ib] : 0;
                    if (va > vb) { out[j] = va; ++ia; } else { out[j] = vb; ++ib; }
                }
            }
            __syncthreads();
            if (active) {
#pragma unroll
                for (int j = 0; j < NP; ++j) lists[threadIdx.x * NP + j] = out[j];
            }
            __syncthreads();
        }
        return;
    }
    uint64_t top[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) top[j] = 0;
    constexpr int kPer = NP <= 4 ? 8 : 2;  // lists per thread per round
    for (uint32_t w0 = 0; w0 < nwarps; w0 += kPer * blockDim.x) {
        uint64_t v[kPer][NP];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const uint32_t w = w0 + u * blockDim.x + threadIdx.x;
            const uint64_t* l = partial + (uint64_t(w < nwarps ? w : 0) * 32 + i) * NP;
#pragma unroll
            for (int j = 0; j < NP; ++j) v[u][j] = w < nwarps ? __ldcg(l + j) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u)
#pragma unroll
            for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, v[u][j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t pv[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) pv[j] = __shfl_xor_sync(0xffffffffu, top[j], o);
#pragma unroll
        for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, pv[j]);
    }
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < NP; ++j) lists[warp * NP + j] = top[j];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int j = 0; j < NP; ++j) top[j] = lane < nw ? lists[lane * NP + j] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t pv[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) pv[j] = __shfl_xor_sync(0xffffffffu, top[j], o);
#pragma unroll
            for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, pv[j]);
        }
    }
    __syncthreads();  // every warp's row of lists was read
    if (threadIdx.x == 0)
#pragma unroll
        for (int j = 0; j < NP; ++j) lists[j] = top[j];
    __syncthreads();
}

template <int NP>
__global__ void topn_merge_kernel(const uint64_t* __restrict__ partial, uint32_t nwarps,
                                  uint32_t nprobe, uint32_t* __restrict__ sel) {
    dev::pdl_wait();
    extern __shared__ uint64_t lists[];  // blockDim x NP
    const uint32_t i = blockIdx.x;
    merge_token_lists<NP>(partial, nwarps, i, lists);
    if (threadIdx.x < nprobe) sel[i * nprobe + threadIdx.x] = dev::key_id(lists[threadIdx.x]);
}

// Candidate generation in one launch (pipeline.cpp:52-87): CTA (i, j) merges
// token i's partial lists (every CTA of the token redundantly — a few tens
// of KB from L2) and ORs the postings of the token's j-th best centroid into
// the N-bit candidate bitmap.
// CTAs past rows x nprobe build stage 2's kept-centroid list (fused::keep_list)
// when `kl` is given: it depends only on the S_cq keep bits, like this kernel.
template <int NP>
__global__ void topn_postings_kernel(const uint64_t* __restrict__ partial, uint32_t nwarps, uint32_t nprobe,
                                     uint32_t ntopn, const uint64_t* __restrict__ ivf_offsets,
                                     const uint32_t* __restrict__ postings, uint32_t* __restrict__ sel,
                                     uint32_t* __restrict__ bitmap, launch::KeepListArgs kl, uint64_t K,
                                     const uint32_t* __restrict__ range_tab, uint32_t range_rows) {
    dev::pdl_wait();
    if (blockIdx.x >= ntopn) {
        fused::keep_list(blockIdx.x - ntopn, gridDim.x - ntopn, kl.keep_bits, K, ivf_offsets, kl.list, kl.counts);
        return;
    }
    extern __shared__ uint64_t lists[];  // blockDim x NP
    const uint32_t i = blockIdx.x / nprobe, j = blockIdx.x % nprobe;
    merge_token_lists<NP>(partial, nwarps, i, lists);
    const uint32_t c = dev::key_id(lists[j]);
    if (threadIdx.x == 0) sel[i * nprobe + j] = c;
    if (!bitmap) {
        // range_stage2 reads the probed lists itself, starting from this
        // centroid's range-table row and list start: warm L2 for it
        if (range_tab) {
            const uint32_t* row = range_tab + uint64_t(c) * range_rows;
            for (uint32_t o = threadIdx.x * 32; o < range_rows; o += blockDim.x * 32)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
            if (threadIdx.x == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(ivf_offsets + c));
        }
        return;
    }
    const uint64_t b = ivf_offsets[c], e = ivf_offsets[c + 1];
    // kU postings per thread in flight: unpredicated loads (index clamped into
    // the list), so the ~2K-entry list costs ~3 HBM round trips, not ~9
    constexpr uint32_t kU = 4;
    for (uint64_t t0 = b + threadIdx.x; t0 < e; t0 += kU * blockDim.x) {
        uint32_t p[kU];
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            const uint64_t t = t0 + u * blockDim.x;
            p[u] = __ldg(postings + (t < e ? t : e - 1));
        }
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u)
            if (t0 + u * blockDim.x < e) atomicOr(bitmap + (p[u] >> 5), 1u << (p[u] & 31));
    }
}

__global__ void token_keys_kernel(const float* __restrict__ S, uint64_t K, uint32_t i,
                                  uint64_t* __restrict__ keys) {
    dev::pdl_wait();
    for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < K;
         c += uint64_t(gridDim.x) * blockDim.x)
        keys[c] = dev::make_key(S[c * kScoresPitch + i], uint32_t(c));
}

__global__ void keys_to_ids_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ n,
                                   uint32_t* __restrict__ ids) {
    dev::pdl_wait();
    const uint64_t cnt = *n;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < cnt;
         j += uint64_t(gridDim.x) * blockDim.x)
        ids[j] = dev::key_id(keys[j]);
}

__global__ void keep_bits_kernel(const float* __restrict__ rowmax, uint64_t K, float t_cs,
                                 uint32_t* __restrict__ bits) {
    dev::pdl_wait();
    const uint64_t words = (K + 31) / 32;
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < words;
         w += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t v = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            uint64_t c = w * 32 + b;
            if (c < K && rowmax[c] >= t_cs) v |= 1u << b;
        }
        bits[w] = v;
    }
}

// Top-NP per query token over a stored S (pipeline.cpp:65-73): warp = a
// contiguous range of centroids, lane = query token, one coalesced 128-byte S
// row per step (8 in flight).  A float bar filters the stream: the lane's own
// NP-th score (strict: later ids lose ties) and a grid-wide bound gthr[token]
// (some warp already holds NP keys scoring >= it, so lower scores cannot reach
// the global top-NP; ties are kept).  Inserts are therefore rare.  Per-warp
// lists go to `partial` for topn_merge.
template <int NP>
__global__ void __launch_bounds__(256)
topn_from_scores_kernel(const float* __restrict__ S, uint64_t K, uint32_t rows, uint64_t* __restrict__ partial,
                        uint32_t* __restrict__ gthr) {
    dev::pdl_wait();
    const uint32_t lane = dev::lane_id();
    const uint64_t gwarp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per = (K + nwarps - 1) / nwarps;
    const uint64_t b = gwarp * per, e = b + per < K ? b + per : K;
    uint64_t top[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) top[j] = 0;
    float thr = -INFINITY, gb = -INFINITY;
    if (lane < rows) {
        for (uint64_t c0 = b; c0 < e; c0 += 8) {
            if (gthr && ((c0 - b) & 63) == 0) {
                const uint32_t go = __ldcg(gthr + lane);
                if (go) gb = dev::unord_f32(go);
            }
            float s[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] = c0 + u < e ? __ldcg(S + (c0 + u) * kScoresPitch + lane) : -INFINITY;
            const float thr0 = thr;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (s[u] > thr && s[u] >= gb) {
                    dev::topn_insert<NP>(top, dev::make_key(s[u], uint32_t(c0 + u)));
                    if (top[NP - 1]) thr = dev::key_score(top[NP - 1]);
                }
            }
            if (gthr && thr > thr0 && thr > gb) {
                atomicMax(gthr + lane, dev::ord_f32(thr));
                gb = thr;
            }
        }
    }
    uint64_t* out = partial + (gwarp * 32 + lane) * NP;
#pragma unroll
    for (int j = 0; j < NP; ++j) out[j] = top[j];
}

__global__ void iota_kernel(uint32_t* __restrict__ out, uint64_t n) {
    dev::pdl_wait();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = uint32_t(i);
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

template <int NP>
void launch_scores(const IndexView& ix, const float* q, uint32_t rows, float t_cs, float* S,
                   float* rowmax, uint32_t* keep, uint64_t* partial, uint32_t blocks,
                   cudaStream_t st) {
    const size_t smem = size_t(32) * (ix.dim + 4) * 4 + size_t(kWarpsPerBlock) * kG * ix.dim * 4;
    static launch::PerDeviceOnce configured;
    if (configured.first()) {
        cudaFuncSetAttribute(scores_exact_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
    }
    ::plaid::launch::pdl(scores_exact_kernel<NP>, blocks, kWarpsPerBlock * 32, smem, st, 
        ix.centroids, ix.K, ix.dim, q, rows, t_cs, S, rowmax, keep, partial);
    launch::count_launch();
}

template <int NP>
void launch_merge(const uint64_t* partial, uint32_t nwarps, uint32_t rows, uint32_t nprobe,
                  uint32_t* sel, cudaStream_t st) {
    const uint32_t threads = 256;
    const size_t smem = threads * NP * sizeof(uint64_t);
    static launch::PerDeviceOnce configured;
    if (configured.first()) {
        cudaFuncSetAttribute(topn_merge_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
    ::plaid::launch::pdl(topn_merge_kernel<NP>, rows, threads, smem, st, partial, nwarps, nprobe, sel);
    launch::count_launch();
}

template <int NP>
void launch_topn_postings(const uint64_t* partial, uint32_t nwarps, uint32_t rows, uint32_t nprobe,
                          const IndexView& ix, uint32_t* sel, uint32_t* bitmap, const launch::KeepListArgs* kl,
                          cudaStream_t st) {
    const uint32_t threads = 256;
    const size_t smem = threads * NP * sizeof(uint64_t);
    static launch::PerDeviceOnce configured;
    if (configured.first()) {
        cudaFuncSetAttribute(topn_postings_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
    const uint32_t ntopn = rows * nprobe;
    const uint32_t nkb = kl ? launch::keep_list_blocks(ix.K) : 0;
    ::plaid::launch::pdl(topn_postings_kernel<NP>, ntopn + nkb, threads, smem, st, partial, nwarps, nprobe, ntopn,
                         ix.ivf_offsets, ix.ivf_postings, sel, bitmap, kl ? *kl : launch::KeepListArgs{}, ix.K,
                         ix.range_tab, ix.range_n + 1);
    launch::count_launch();
}

}  // namespace

namespace launch {

uint32_t scores_max_warps() { return uint32_t(sm_count()) * kBlocksPerSm * kWarpsPerBlock; }

uint32_t scores_exact(const IndexView& ix, const float* d_q, uint32_t rows, float t_cs,
                      float* d_scores, float* d_rowmax, uint32_t* d_keep_bits, uint64_t* d_partial,
                      uint32_t np_bucket, cudaStream_t st) {
    const uint64_t chunks = (ix.K + 31) / 32;
    uint64_t want = (chunks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    uint32_t blocks = uint32_t(want < uint64_t(sm_count()) * kBlocksPerSm ? want
                                                                          : uint64_t(sm_count()) * kBlocksPerSm);
    if (blocks == 0) blocks = 1;
    switch (np_bucket) {
        case 1: launch_scores<1>(ix, d_q, rows, t_cs, d_scores, d_rowmax, d_keep_bits, d_partial, blocks, st); break;
        case 2: launch_scores<2>(ix, d_q, rows, t_cs, d_scores, d_rowmax, d_keep_bits, d_partial, blocks, st); break;
        case 4: launch_scores<4>(ix, d_q, rows, t_cs, d_scores, d_rowmax, d_keep_bits, d_partial, blocks, st); break;
        case 8: launch_scores<8>(ix, d_q, rows, t_cs, d_scores, d_rowmax, d_keep_bits, d_partial, blocks, st); break;
        case 16: launch_scores<16>(ix, d_q, rows, t_cs, d_scores, d_rowmax, d_keep_bits, d_partial, blocks, st); break;
        default: launch_scores<32>(ix, d_q, rows, t_cs, d_scores, d_rowmax, d_keep_bits, d_partial, blocks, st); break;
    }
    return blocks * kWarpsPerBlock;
}

void topn_postings(const uint64_t* d_partial, uint32_t num_warps, uint32_t np_bucket, uint32_t rows, uint32_t nprobe,
                   const IndexView& ix, uint32_t* d_sel, uint32_t* d_bitmap, const KeepListArgs* kl,
                   cudaStream_t st) {
    switch (np_bucket) {
        case 1: launch_topn_postings<1>(d_partial, num_warps, rows, nprobe, ix, d_sel, d_bitmap, kl, st); break;
        case 2: launch_topn_postings<2>(d_partial, num_warps, rows, nprobe, ix, d_sel, d_bitmap, kl, st); break;
        case 4: launch_topn_postings<4>(d_partial, num_warps, rows, nprobe, ix, d_sel, d_bitmap, kl, st); break;
        case 8: launch_topn_postings<8>(d_partial, num_warps, rows, nprobe, ix, d_sel, d_bitmap, kl, st); break;
        case 16: launch_topn_postings<16>(d_partial, num_warps, rows, nprobe, ix, d_sel, d_bitmap, kl, st); break;
        default: launch_topn_postings<32>(d_partial, num_warps, rows, nprobe, ix, d_sel, d_bitmap, kl, st); break;
    }
}

void topn_merge(const uint64_t* d_partial, uint32_t num_warps, uint32_t np_bucket, uint32_t rows,
                uint32_t nprobe, uint32_t* d_sel, cudaStream_t st) {
    switch (np_bucket) {
        case 1: launch_merge<1>(d_partial, num_warps, rows, nprobe, d_sel, st); break;
        case 2: launch_merge<2>(d_partial, num_warps, rows, nprobe, d_sel, st); break;
        case 4: launch_merge<4>(d_partial, num_warps, rows, nprobe, d_sel, st); break;
        case 8: launch_merge<8>(d_partial, num_warps, rows, nprobe, d_sel, st); break;
        case 16: launch_merge<16>(d_partial, num_warps, rows, nprobe, d_sel, st); break;
        default: launch_merge<32>(d_partial, num_warps, rows, nprobe, d_sel, st); break;
    }
}

void token_keys(const float* d_scores, uint64_t K, uint32_t i, uint64_t* d_keys, cudaStream_t st) {
    uint64_t blocks = (K + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    ::plaid::launch::pdl(token_keys_kernel, uint32_t(blocks), 256, 0, st, d_scores, K, i, d_keys);
    count_launch();
}

void keys_to_ids(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint32_t* d_ids,
                 cudaStream_t st) {
    uint64_t blocks = (nmax + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks == 0) blocks = 1;
    ::plaid::launch::pdl(keys_to_ids_kernel, uint32_t(blocks), 256, 0, st, d_keys, d_n, d_ids);
    count_launch();
}

void keep_bits_from_rowmax(const float* d_rowmax, uint64_t K, float t_cs, uint32_t* d_keep_bits,
                           cudaStream_t st) {
    uint64_t words = (K + 31) / 32;
    uint64_t blocks = (words + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    ::plaid::launch::pdl(keep_bits_kernel, uint32_t(blocks), 256, 0, st, d_rowmax, K, t_cs, d_keep_bits);
    count_launch();
}

uint32_t topn_from_scores(const float* d_scores, uint64_t K, uint32_t rows, uint64_t* d_partial,
                          uint32_t np_bucket, uint32_t* d_gthr, cudaStream_t st) {
    const uint32_t blocks = uint32_t(sm_count()) * kBlocksPerSm;
    const uint32_t threads = kWarpsPerBlock * 32;
    switch (np_bucket) {
        case 1: ::plaid::launch::pdl(topn_from_scores_kernel<1>, blocks, threads, 0, st, d_scores, K, rows, d_partial, d_gthr); break;
        case 2: ::plaid::launch::pdl(topn_from_scores_kernel<2>, blocks, threads, 0, st, d_scores, K, rows, d_partial, d_gthr); break;
        case 4: ::plaid::launch::pdl(topn_from_scores_kernel<4>, blocks, threads, 0, st, d_scores, K, rows, d_partial, d_gthr); break;
        case 8: ::plaid::launch::pdl(topn_from_scores_kernel<8>, blocks, threads, 0, st, d_scores, K, rows, d_partial, d_gthr); break;
        case 16: ::plaid::launch::pdl(topn_from_scores_kernel<16>, blocks, threads, 0, st, d_scores, K, rows, d_partial, d_gthr); break;
        default: ::plaid::launch::pdl(topn_from_scores_kernel<32>, blocks, threads, 0, st, d_scores, K, rows, d_partial, d_gthr); break;
    }
    count_launch();
    return blocks * kWarpsPerBlock;
}

void iota(uint32_t* d_out, uint64_t n, cudaStream_t st) {
    uint64_t b = (n + 255) / 256;
    ::plaid::launch::pdl(iota_kernel, uint32_t(b > 4096 ? 4096 : (b ? b : 1)), 256, 0, st, d_out, n);
    count_launch();
}

}  // namespace launch
}  // namespace plaid
