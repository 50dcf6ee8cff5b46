// select.cu — select_top (pipeline.cpp:139-163) on 64-bit keys.
//
// Keys pack (ord(score) << 32 | ~id), so "largest key first" is exactly the
// reference's (score desc, id asc) order and every key is unique.  Two paths:
//   * select_top_large: ONE cooperative kernel doing an MSB radix select over
//     the 64-bit keys (digit passes of 11,11,11,11,11,9 bits; a grid barrier
//     after each pass, then every CTA derives the same digit from the global
//     histogram, so there is no host round trip and no extra launch), then a
//     compaction of the keys >= the threshold (unordered).  Used for stage 2,
//     whose input is the whole candidate set.
//   * sort_top: one CTA bitonic sort in shared memory (<= 8192 keys; one
//     comparator per thread per step), or a global-memory bitonic network
//     beyond that; emits the first `want` keys as (id, score) pairs in order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device.cuh"
#include "fused.cuh"
#include "kernels.cuh"
#include "s4_mma.cuh"

namespace plaid {
namespace {

constexpr uint32_t kBins = 2048;
constexpr int kPasses = 6;
constexpr uint32_t kSelThreads = 512;
constexpr uint32_t kBoundaryCap = 1024;  // boundary-bucket keys resolved in one CTA (fits h[] as u64)
static_assert(kBoundaryCap * 8 <= kBins * 4, "boundary keys reuse the histogram's shared memory");
__host__ __device__ constexpr int pass_shift(int p) { return p < 5 ? 53 - 11 * p : 0; }
__host__ __device__ constexpr int pass_bits(int p) { return p < 5 ? 11 : 9; }

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).
__device__ __forceinline__ void grid_sync(unsigned int* count, unsigned int* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* vgen = gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads)
radix_select_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n, uint64_t want,
                    SelectState* st, uint64_t* __restrict__ out, uint64_t* __restrict__ out_n) {
    dev::pdl_wait();
    __shared__ __align__(16) uint32_t h[kBins];
    __shared__ uint32_t part[kSelThreads];
    __shared__ unsigned long long s_prefix, s_mask, s_rem;
    __shared__ int s_done, s_small;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const uint64_t n = *d_n;
    if (tid == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_rem = n < want ? n : want;
        s_done = n <= want;
        s_small = 0;
    }
    const uint64_t stride = uint64_t(gridDim.x) * kSelThreads;
    for (int pass = 0; pass < kPasses; ++pass) {
        __syncthreads();
        if (s_done || s_small) break;
        const int shift = pass_shift(pass);
        const uint32_t nb = 1u << pass_bits(pass);
        const uint64_t prefix = s_prefix, mask = s_mask;
        for (uint32_t b = tid; b < nb; b += kSelThreads) h[b] = 0;
        __syncthreads();
        for (uint64_t i0 = uint64_t(blockIdx.x) * kSelThreads; i0 < n; i0 += stride) {
            const uint64_t i = i0 + tid;
            const uint64_t k = i < n ? __ldcg(keys + i) : 0;
            const bool valid = i < n && (k & mask) == prefix;
            const uint32_t bin = valid ? uint32_t(k >> shift) & (nb - 1) : 0xFFFFFFFFu;
            // warp-aggregated: the many equal keys of a dense bucket (e.g. the
            // all-masked zero scores of stage 2) cost one atomic per warp
            const uint32_t peers = __match_any_sync(0xffffffffu, bin);
            if (valid && lane == uint32_t(__ffs(peers) - 1)) atomicAdd(&h[bin], uint32_t(__popc(peers)));
        }
        __syncthreads();
        for (uint32_t b = tid; b < nb; b += kSelThreads)
            if (h[b]) atomicAdd(&st->hist[pass][b], h[b]);
        grid_sync(&st->bar_count, &st->bar_gen);
        // every CTA: the bin (from the top) holding the s_rem-th largest key
        const uint32_t per = nb / kSelThreads;  // 4 or 1
        uint32_t mine = 0;
        for (uint32_t j = 0; j < per; ++j) mine += __ldcg(&st->hist[pass][nb - 1 - (tid * per + j)]);
        // block inclusive scan of `mine` (descending-bin order)
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += v;
        }
        if (lane == 31) part[tid >> 5] = incl;
        __syncthreads();
        uint32_t before = 0;
        for (uint32_t w = 0; w < (tid >> 5); ++w) before += part[w];
        const uint64_t cum0 = uint64_t(before) + incl - mine;  // keys in bins above mine
        const uint64_t rem = s_rem;
        __syncthreads();
        if (cum0 < rem && rem <= cum0 + mine) {
            uint64_t cum = cum0;
            for (uint32_t j = 0; j < per; ++j) {
                const uint32_t bin = nb - 1 - (tid * per + j);
                const uint32_t cnt = __ldcg(&st->hist[pass][bin]);
                if (cum + cnt >= rem) {
                    s_rem = rem - cum;
                    s_prefix = prefix | (uint64_t(bin) << shift);
                    s_mask = mask | (uint64_t(nb - 1) << shift);
                    s_done = cnt == rem - cum;
                    // a small boundary bucket is resolved exactly in one CTA
                    // instead of by further passes over all n keys
                    s_small = cnt <= kBoundaryCap;
                    break;
                }
                cum += cnt;
            }
        }
    }
    __syncthreads();
    if (s_small && !s_done) {
        // keys above the boundary bucket are all in; the bucket's keys (at
        // most kBoundaryCap) go to st->bnd and CTA 0 keeps their top s_rem
        const uint64_t prefix = s_prefix, mask = s_mask;
        for (uint64_t i0 = uint64_t(blockIdx.x) * kSelThreads; i0 < n; i0 += stride) {
            const uint64_t i = i0 + tid;
            const uint64_t k = i < n ? __ldcg(keys + i) : 0;
            const uint64_t top = k & mask;
            const bool above = i < n && top > prefix, inb = i < n && top == prefix;
            const uint32_t ba = __ballot_sync(0xffffffffu, above), bb = __ballot_sync(0xffffffffu, inb);
            if (ba) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd((unsigned long long*)out_n, (unsigned long long)__popc(ba));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (above) out[base + __popc(ba & ((1u << lane) - 1))] = k;
            }
            if (bb) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&st->bnd_n, uint32_t(__popc(bb)));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (inb) st->bnd[base + __popc(bb & ((1u << lane) - 1))] = k;
            }
        }
        grid_sync(&st->bar_count, &st->bar_gen);
        if (blockIdx.x != 0) return;
        unsigned long long* sb = reinterpret_cast<unsigned long long*>(h);  // kBins u32 = kBoundaryCap u64
        const uint32_t nbd = __ldcg(&st->bnd_n);
        for (uint32_t j = tid; j < nbd; j += kSelThreads) sb[j] = __ldcg(&st->bnd[j]);
        __syncthreads();
        const uint64_t rem = s_rem;
        for (uint32_t j = tid; j < nbd; j += kSelThreads) {
            const unsigned long long x = sb[j];
            uint32_t rank = 0;
            for (uint32_t m = 0; m < nbd; ++m) rank += sb[m] > x;
            if (rank < rem) out[atomicAdd((unsigned long long*)out_n, 1ull)] = x;
        }
        return;
    }
    // compaction of every key >= threshold (exactly min(want, n) keys)
    const uint64_t thr = s_prefix;
    for (uint64_t i0 = uint64_t(blockIdx.x) * kSelThreads; i0 < n; i0 += stride) {
        const uint64_t i = i0 + tid;
        const uint64_t k = i < n ? __ldcg(keys + i) : 0;
        const bool take = i < n && k >= thr;
        const uint32_t ballot = __ballot_sync(0xffffffffu, take);
        if (!ballot) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd((unsigned long long*)out_n, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) out[base + __popc(ballot & ((1u << lane) - 1))] = k;
    }
}

// Emit the j-th key of a descending array.
__device__ __forceinline__ void emit(uint64_t j, uint64_t key, uint64_t* out_keys, uint32_t* out_ids,
                                     float* out_scores, uint32_t id_base) {
    if (out_keys) out_keys[j] = key;
    if (out_ids) out_ids[j] = dev::key_id(key) + id_base;
    if (out_scores) out_scores[j] = dev::key_score(key);
}

// Bitonic network step over s[0..npad): comparator p (< npad/2) joins
// i = insert a 0 bit at position log2(j) of p, and i + j.
__device__ __forceinline__ void bitonic_pair(uint64_t* s, uint32_t p, uint32_t j, uint32_t k) {
    const uint32_t i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
    const uint32_t ixj = i + j;
    const uint64_t a = s[i], b = s[ixj];
    const bool desc = (i & k) == 0;
    if (desc ? (a < b) : (a > b)) {
        s[i] = b;
        s[ixj] = a;
    }
}

__global__ void __launch_bounds__(1024)
sort_small_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n, uint32_t npad,
                  uint64_t want, uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_ids,
                  float* __restrict__ out_scores, uint64_t* __restrict__ out_n, uint32_t id_base) {
    dev::pdl_wait();
    extern __shared__ uint64_t s[];
    const uint64_t n = *d_n;
    for (uint32_t i = threadIdx.x; i < npad; i += blockDim.x) s[i] = i < n ? keys[i] : 0ull;
    __syncthreads();
    const uint32_t half = npad >> 1;
    for (uint32_t k = 2; k <= npad; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t p = threadIdx.x; p < half; p += blockDim.x) bitonic_pair(s, p, j, k);
            __syncthreads();
        }
    }
    const uint64_t m = n < want ? n : want;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) emit(j, s[j], out_keys, out_ids, out_scores, id_base);
    if (threadIdx.x == 0 && out_n) *out_n = m;
}

// Sort by rank (n <= kSmallSortMax): keys are unique, so the position of key
// x in the descending order is the number of keys greater than x.  Every CTA
// stages all n keys in shared memory and each thread ranks one key against
// them (broadcast reads, two keys per 128-bit load); keys with rank < want
// are written straight to their slot.  O(n^2) compares, but spread over the
// whole GPU it beats a single-CTA bitonic network (78 barrier-separated
// steps at n = 4096) by an order of magnitude.
// A CTA ranks 32 keys with 4 threads each (thread q of a key scans quarter q
// of the array); quarters start one 16-byte pair apart in bank space, so the
// four addresses of a warp-wide load never share a bank.
constexpr uint32_t kRankThreads = 128;
constexpr uint32_t kRankPerCta = kRankThreads / 4;

__host__ __device__ constexpr uint32_t rank_quarter_pairs(uint32_t n) {
    return (((n + 1) / 2 + 3) / 4 + 7) / 8 * 8;  // pairs per quarter, a multiple of 8
}

__global__ void __launch_bounds__(kRankThreads)
sort_rank_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n, uint64_t want,
                 uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_ids, float* __restrict__ out_scores,
                 uint64_t* __restrict__ out_n, uint32_t id_base) {
    dev::pdl_wait();
    extern __shared__ __align__(16) uint64_t s[];
    const uint32_t n = uint32_t(*d_n);
    if (blockIdx.x == 0 && threadIdx.x == 0 && out_n) *out_n = n < want ? n : want;
    if (blockIdx.x * kRankPerCta >= n) return;
    const uint32_t npq = rank_quarter_pairs(n);
    // pair k of quarter q lives at pair slot q * (npq + 1) + k
    for (uint32_t i = threadIdx.x; i < 4 * (npq + 1); i += kRankThreads) {
        const uint32_t q = i / (npq + 1), k = i % (npq + 1);
        const uint32_t e = 2 * (q * npq + k);
        const bool real = k < npq;
        s[2 * i] = real && e < n ? __ldcg(keys + e) : 0ull;
        s[2 * i + 1] = real && e + 1 < n ? __ldcg(keys + e + 1) : 0ull;
    }
    __syncthreads();
    const uint32_t me = blockIdx.x * kRankPerCta + (threadIdx.x >> 2), q = threadIdx.x & 3;
    const uint64_t x = me < n ? __ldcg(keys + me) : ~0ull;
    uint32_t rank = 0;
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(s) + q * (npq + 1);
#pragma unroll 8
    for (uint32_t j = 0; j < npq; ++j) {
        const ulonglong2 v = s2[j];
        rank += (v.x > x) + (v.y > x);
    }
    rank += __shfl_xor_sync(0xffffffffu, rank, 1);
    rank += __shfl_xor_sync(0xffffffffu, rank, 2);
    if (q == 0 && me < n && rank < want) emit(rank, x, out_keys, out_ids, out_scores, id_base);
}

// Stage 4's last two launches in one (finalize_kernel + sort_rank_kernel):
// every CTA sums the running maxima of ALL n finalists itself (n x 128 B of
// `run`, L2-resident after stage 4; the same in-order fp32 adds as
// finalize_kernel, rank128.cu) into a shared-memory key array, thread per
// finalist so that every row load of the CTA is in flight at once, then warp
// w ranks key 32 b + w (lane j counts the keys j, j + 32, ... above it).  The
// redundant reads (n x 128 B per CTA, one L2 round trip) cost less than the
// launch boundary they remove.  `run` must be zero again for the next stage
// 4: the last CTA done reading it (a ticket counter, zero at launch) clears
// the n rows.
constexpr uint32_t kFinRankThreads = 1024;
constexpr uint32_t kFinRankPerCta = kFinRankThreads / 32;
constexpr uint32_t kFinTileWords = (kFinRankThreads / 32) * 32 * 33;  // one 32 x 33 float tile per warp
__global__ void __launch_bounds__(kFinRankThreads)
finalize_rank_kernel(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ fkeys,
                     const uint64_t* __restrict__ d_n, uint32_t rows, uint32_t* __restrict__ run, uint64_t want,
                     uint32_t* __restrict__ out_ids, float* __restrict__ out_scores, uint64_t* __restrict__ out_n,
                     uint32_t id_base, unsigned int* __restrict__ ticket) {
    dev::pdl_wait();
    extern __shared__ __align__(16) uint64_t sm[];
    uint64_t* s = sm + kFinTileWords / 2;  // keys after the warps' tiles
    __shared__ uint32_t s_last;
    const uint32_t n = uint32_t(*d_n);
    if (blockIdx.x == 0 && threadIdx.x == 0 && out_n) *out_n = n < want ? n : want;
    // warp w takes rows [32 r, 32 r + 32) for r = w, w + 32, ...: coalesced
    // 512-byte loads (4 rows per instruction) into a per-warp 32 x 33 tile,
    // then lane = row: the in-order sum.  (A thread reading its own 128-byte
    // row would touch 32 lines per instruction: 8 K L1 wavefronts per CTA.)
    float* tile = reinterpret_cast<float*>(sm) + (threadIdx.x >> 5) * 32 * 33;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t r0 = (threadIdx.x >> 5) * 32; r0 < n; r0 += kFinRankThreads) {
        const uint4* r4 = reinterpret_cast<const uint4*>(run + uint64_t(r0) * 32);
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t row = 4 * j + lane / 8;
            v[j] = r0 + row < n ? __ldcg(r4 + 32 * j + lane) : make_uint4(0, 0, 0, 0);
        }
        const uint32_t e = r0 + lane;
        const uint32_t pid = e < n ? (ids ? __ldcg(ids + e) : dev::key_id(__ldcg(fkeys + e))) : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float* t = tile + (4 * j + lane / 8) * 33 + (lane % 8) * 4;
            t[0] = dev::unord_f32(v[j].x), t[1] = dev::unord_f32(v[j].y);
            t[2] = dev::unord_f32(v[j].z), t[3] = dev::unord_f32(v[j].w);
        }
        __syncwarp();
        float total = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (uint32_t(i) < rows) total = __fadd_rn(total, tile[lane * 33 + i]);
        if (e < n) s[e] = dev::make_key(total, pid);
        __syncwarp();
    }
    __syncthreads();  // this CTA's reads of `run` are complete
    // the ticket's round trip overlaps the ranking: issued here, its value
    // first needed after the emit
    unsigned int tk = 0;
    if (threadIdx.x == 0)
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(tk) : "l"(ticket) : "memory");
    const uint32_t me = blockIdx.x * kFinRankPerCta + (threadIdx.x >> 5);
    if (me < n) {
        const uint64_t x = s[me];
        uint32_t rank = 0;
#pragma unroll 4
        for (uint32_t j = lane; j < n; j += 32) rank += s[j] > x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
        if (lane == 0 && rank < want) emit(rank, x, nullptr, out_ids, out_scores, id_base);
    }
    if (threadIdx.x == 0) s_last = tk == gridDim.x - 1;
    __syncthreads();
    if (s_last) {  // every CTA has read `run`: clear it for the next stage 4
        uint4* r4 = reinterpret_cast<uint4*>(run);
        for (uint32_t i = threadIdx.x; i < n * 8; i += kFinRankThreads) r4[i] = make_uint4(0, 0, 0, 0);
    }
}

__global__ void pad_copy_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                                uint64_t npad, uint64_t* __restrict__ tmp) {
    dev::pdl_wait();
    const uint64_t n = *d_n;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < npad;
         i += uint64_t(gridDim.x) * blockDim.x)
        tmp[i] = i < n ? keys[i] : 0ull;
}

__global__ void bitonic_step_kernel(uint64_t* __restrict__ s, uint64_t npad, uint64_t j, uint64_t k) {
    dev::pdl_wait();
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < npad / 2;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
        const uint64_t ixj = i + j;
        const uint64_t a = s[i], b = s[ixj];
        const bool desc = (i & k) == 0;
        if (desc ? (a < b) : (a > b)) {
            s[i] = b;
            s[ixj] = a;
        }
    }
}

__global__ void emit_kernel(const uint64_t* __restrict__ sorted, const uint64_t* __restrict__ d_n,
                            uint64_t want, uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_ids,
                            float* __restrict__ out_scores, uint64_t* __restrict__ out_n, uint32_t id_base) {
    dev::pdl_wait();
    const uint64_t n = *d_n;
    const uint64_t m = n < want ? n : want;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < m;
         j += uint64_t(gridDim.x) * blockDim.x)
        emit(j, sorted[j], out_keys, out_ids, out_scores, id_base);
    if (blockIdx.x == 0 && threadIdx.x == 0 && out_n) *out_n = m;
}

__global__ void make_keys_kernel(const uint32_t* __restrict__ ids, const float* __restrict__ scores,
                                 uint64_t n, uint64_t* __restrict__ keys) {
    dev::pdl_wait();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        keys[i] = dev::make_key(scores[i], ids[i]);
}

// Per shard g, entries [0, counts[g]) of row g (stride) become keys; the rest
// of the G*stride slots are 0 (below every real key).
// (rows may be packed: shard g's pids at pids + g * stride, its count at
// counts[g * count_stride]; only the first `k` entries of a row are read)
__global__ void merge_keys_kernel(const uint32_t* __restrict__ pids, const float* __restrict__ scores,
                                  const uint64_t* __restrict__ counts, uint64_t shards, uint64_t stride,
                                  uint64_t count_stride, uint64_t k, uint64_t* __restrict__ keys,
                                  uint64_t* __restrict__ d_n) {
    dev::pdl_wait();
    const uint64_t total = shards * k;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = i / k, j = i % k;
        const uint64_t at = g * stride + j;
        keys[i] = j < counts[g * count_stride] ? dev::make_key(scores[at], pids[at]) : 0ull;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *d_n = total;
}

__global__ void copy_count_kernel(const uint64_t* src, uint64_t* dst, uint64_t cap) {
    dev::pdl_wait();
    const uint64_t v = *src;
    *dst = v < cap ? v : cap;
}

// Per-query prologue, one PDL-chained launch instead of a memset plus a
// validation kernel: every CTA zeroes its share of the per-query counters and
// bitmaps; when q != nullptr the last CTA also checks the query rows
// (check_unit_rows, types.cpp:10-19: norm^2 = sum of double(v)^2 in order —
// the products are exact in fp64, so only the adds must stay in order).
// bf16 bits of x rounded to nearest even (finite inputs)
__device__ __forceinline__ uint32_t bf16_rn_u32(float x) {
    const uint32_t u = __float_as_uint(x);
    return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

// The stage-4 tensor kernel's B operand for a query (rank128.cu,
// stage4_tensor_kernel): 64 rows x K = 256 bf16, row n < 32 = [Q_hi | Q_hi]
// of query token n, row 32 + i = [Q_lo | 0] of token i (Q_hi = bf16(q),
// Q_lo = bf16(q - Q_hi); zero rows past `rows`), SWIZZLE_128B K-major chunks
// of 64 bf16: chunk c, row n, 16-byte granule j at c * 8192 + n * 128 +
// ((j ^ (n & 7)) << 4).
// One 16-byte granule e of the image (e < kQImgBytes / 16).
__device__ __forceinline__ void qimg_granule(const float* __restrict__ q, uint32_t rows, uint32_t e,
                                             uint4* __restrict__ img) {
    const uint32_t c = e >> 9, n = (e >> 3) & 63, j = e & 7;
    const uint32_t i = n & 31, k0 = c * 64 + j * 8, d0 = k0 & 127;
    const bool lo = n >= 32;
    uint32_t v[4] = {0, 0, 0, 0};
    if (i < rows && !(lo && k0 >= 128)) {
        const float4 a = reinterpret_cast<const float4*>(q + i * 128 + d0)[0];
        const float4 b = reinterpret_cast<const float4*>(q + i * 128 + d0)[1];
        const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint32_t h0 = bf16_rn_u32(f[2 * u]), h1 = bf16_rn_u32(f[2 * u + 1]);
            if (lo) {
                h0 = bf16_rn_u32(f[2 * u] - __uint_as_float(h0 << 16));
                h1 = bf16_rn_u32(f[2 * u + 1] - __uint_as_float(h1 << 16));
            }
            v[u] = h0 | (h1 << 16);
        }
    }
    img[(c * 8192 + n * 128 + ((j ^ (n & 7)) << 4)) / 16] = make_uint4(v[0], v[1], v[2], v[3]);
}

// Every piece of the prologue is spread over the whole grid (one element per
// thread), so none of it is a serial chain of round trips on one CTA: the
// query rows may sit in pinned host memory (host path), where each dependent
// load costs a PCIe round trip, and the S_cq kernel waits for this grid.
__global__ void __launch_bounds__(256) query_prologue_kernel(const float* __restrict__ q, uint32_t rows, uint32_t dim,
                                                              int* __restrict__ status, uint4* __restrict__ zero,
                                                              uint64_t n16, uint4* __restrict__ zero2, uint64_t m16,
                                                              const float* __restrict__ qsrc, uint4* __restrict__ qimg,
                                                              float* __restrict__ qcopy, uint32_t ncopy4) {
    dev::pdl_wait();
    // let the S_cq kernel launch now: its TMA producer streams the centroid
    // table (no dependence on this kernel) while the zero fill runs; its other
    // warps still wait for this grid to complete
    dev::pdl_trigger();
    // with validation the last CTA only runs the norm check (its serial fp64
    // chains then overlap the other CTAs' work instead of following its own)
    const bool checker = q != nullptr && blockIdx.x == gridDim.x - 1;
    const uint32_t work_ctas = q != nullptr ? gridDim.x - 1 : gridDim.x;
    const uint64_t gt = checker ? ~0ull : blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint64_t nt = uint64_t(work_ctas) * blockDim.x;
    // host path: the query rows come straight from the caller's pinned
    // (mapped) staging buffer — no separate H2D copy ahead of this kernel
    if (qcopy)
        for (uint64_t i = gt; i < ncopy4; i += nt)
            reinterpret_cast<float4*>(qcopy)[i] = reinterpret_cast<const float4*>(qsrc)[i];
    if (qimg) {
        for (uint64_t e = gt; e < launch::kQImgBytes / 16; e += nt) qimg_granule(qsrc, rows, uint32_t(e), qimg);
        // the mma.sync B fragments (s4_mma.cuh) after it
        uint2* qf = reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(qimg) + launch::kQImgBytes);
        for (uint64_t e = gt; e < 8 * 4 * 32; e += nt) {
            const uint32_t ln = uint32_t(e) & 31, j = (uint32_t(e) >> 5) & 3, ks = uint32_t(e) >> 7;
            const uint32_t n = 8 * j + (ln >> 2), k0 = 16 * ks + 2 * (ln & 3);
            float x[4] = {0.f, 0.f, 0.f, 0.f};
            if (n < rows) {
                const float* qr = qsrc + uint64_t(n) * 128 + k0;
                x[0] = qr[0], x[1] = qr[1], x[2] = qr[8], x[3] = qr[9];
            }
            qf[((ks * 4 + j) * 2 + 0) * 32 + ln] = make_uint2(s4mma::bf16_pair(x[0], x[1]), s4mma::bf16_pair(x[2], x[3]));
            qf[((ks * 4 + j) * 2 + 1) * 32 + ln] =
                make_uint2(s4mma::bf16_pair_lo(x[0], x[1]), s4mma::bf16_pair_lo(x[2], x[3]));
        }
    }
    for (uint64_t i = gt; i < n16 + m16; i += nt) {
        if (i < n16) zero[i] = make_uint4(0, 0, 0, 0);
        else zero2[i - n16] = make_uint4(0, 0, 0, 0);
    }
    // the norm check of row r (check_unit_rows, types.cpp:10-19) in the last
    // CTA: 128-dim slabs of all rows staged with one coalesced round of loads,
    // then thread r runs row r's in-order fp64 add chain from shared memory
    // (the squares are exact in fp64)
    if (!checker) return;
    __shared__ float slab[32][129];
    double acc = 0.0;
    for (uint32_t d0 = 0; d0 < dim; d0 += 128) {
        const uint32_t w = dim - d0 < 128 ? dim - d0 : 128;
        float v[16];  // 32 x 128 / 256 threads: every load in flight at once
#pragma unroll
        for (uint32_t k = 0; k < 16; ++k) {
            const uint32_t i = threadIdx.x + k * 256, r = i >> 7, d = i & 127;
            v[k] = r < rows && d < w ? q[size_t(r) * dim + d0 + d] : 0.f;
        }
#pragma unroll
        for (uint32_t k = 0; k < 16; ++k) {
            const uint32_t i = threadIdx.x + k * 256;
            slab[i >> 7][i & 127] = v[k];
        }
        __syncthreads();
        if (threadIdx.x < rows)
            for (uint32_t d = 0; d < w; ++d) {
                const double v = double(slab[threadIdx.x][d]);
                acc = __dadd_rn(acc, __dmul_rn(v, v));
            }
        __syncthreads();
    }
    if (threadIdx.x >= rows) return;
    const double norm = sqrt(acc);
    if (fabs(norm - 1.0) > double(1e-3f)) atomicExch(status, 2);  // NotNormalized + 1
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

uint32_t grid_for(uint64_t n, uint32_t threads, uint32_t cap) {
    uint64_t b = (n + threads - 1) / threads;
    if (b > cap) b = cap;
    return uint32_t(b ? b : 1);
}

uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

// ---- histogram select (no grid barriers) ----------------------------------------------
constexpr uint32_t kHistBucketShift = kHistShift;

// The bucket (from the top) holding the want-th largest key, found by every
// CTA of the compaction for itself (no separate single-CTA launch): the 32
// block sums SelectHist::blk (one L2 round trip) give the block, then thread t
// sums buckets [8 t, 8 t + 8) of that block (one more round trip) and a
// block-wide suffix scan gives the bucket (threads 0-255 hold the buckets).
struct HistBoundary {
    unsigned long long above, bcount, rem;
    uint32_t bucket, take_all;
};

__device__ __forceinline__ void hist_boundary(const SelectHist* __restrict__ st, uint64_t n, uint64_t want,
                                              HistBoundary& hb /* shared */) {
    __shared__ unsigned long long blk_above;
    __shared__ uint32_t blk_id, wsum[8];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {  // defaults select nothing should the sums ever disagree with n
        blk_id = 0, blk_above = 0;
        hb.take_all = 0, hb.bucket = 0xFFFFFFFFu, hb.above = 0, hb.bcount = 0, hb.rem = 0;
    }
    __syncthreads();
    if (n <= want) {
        if (t == 0) hb.take_all = 1, hb.bucket = 0, hb.above = 0, hb.bcount = 0, hb.rem = 0;
        __syncthreads();
        return;
    }
    if (warp == 0) {
        const uint32_t c = __ldcg(&st->blk[lane]);
        // inclusive suffix sum: keys in blocks >= lane (higher blocks = higher keys)
        unsigned long long incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_down_sync(0xffffffffu, incl, o);
            if (lane + o < 32) incl += y;
        }
        if (incl >= want && incl - c < want) blk_id = lane, blk_above = incl - c;
    }
    __syncthreads();
    const uint32_t B = blk_id;
    uint32_t v[8], mine = 0;  // threads >= 256 (wider CTAs) hold no buckets
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        v[j] = t < 256 ? __ldcg(&st->hist[dev::hist_slot(B * 2048 + 8 * t + j)]) : 0u;
        mine += v[j];
    }
    // suffix scan over the 256 threads (thread 255 holds the top buckets)
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += y;
    }
    if (lane == 0 && warp < 8) wsum[warp] = incl;
    __syncthreads();
    unsigned long long above = blk_above;
    for (uint32_t w = warp + 1; w < 8; ++w) above += wsum[w];
    above += incl - mine;  // keys in this block above thread t's buckets
    if (above < want && want <= above + mine) {
        for (int j = 7; j >= 0; --j) {
            if (above + v[j] >= want) {
                hb.take_all = 0;
                hb.bucket = B * 2048 + 8 * t + uint32_t(j);
                hb.above = above;
                hb.bcount = v[j];
                hb.rem = want - above;
                break;
            }
            above += v[j];
        }
    }
    __syncthreads();
}

// The top `rem` keys of the boundary bucket (keys are unique) appended to
// out, by one CTA of kHistThreads: an MSB-first 8-bit radix select over the
// low 48 bits (the bucket fixes the top 16), each digit found by a
// warp-parallel suffix scan of the 256 counts, stopping early once the
// digit's whole bucket is taken; then every key >= the threshold is written.
// `src` is shared memory (small buckets, staged) or global memory.
constexpr uint32_t kHistThreads = 1024;
constexpr uint32_t kResolveStage = 16384;  // boundary buckets staged in shared memory (dynamic) up to this size
__device__ void resolve_bucket_cta(const uint64_t* src, uint32_t nb, uint64_t rem, uint32_t bucket,
                                   uint64_t* __restrict__ out, uint64_t* __restrict__ out_n) {
    __shared__ uint32_t h[256];
    __shared__ unsigned long long s_prefix, s_rem;
    __shared__ uint32_t s_done;
    const uint32_t t = threadIdx.x, lane = t & 31;
    if (t == 0) s_prefix = 0, s_rem = rem, s_done = 0;
    uint64_t mask = 0;
    for (int shift = 40; shift >= 0; shift -= 8) {
        if (t < 256) h[t] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (uint32_t i = t; i < nb; i += kHistThreads) {
            const uint64_t k = src[i] & 0xFFFFFFFFFFFFull;
            if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (t < 32) {  // lane l: digits 255 - 8 l .. 248 - 8 l, suffix sums from the top
            uint32_t c[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) sum += (c[j] = h[255 - 8 * lane - j]);
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= uint32_t(o)) incl += y;
            }
            const uint64_t r = s_rem;
            uint64_t above = incl - sum;
            if (above < r && r <= above + sum) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (above < r && r <= above + c[j]) {
                        s_prefix = prefix | (uint64_t(255 - 8 * lane - j) << shift);
                        s_rem = r - above;
                        s_done = c[j] == r - above;  // the digit's whole bucket is taken
                    }
                    above += c[j];
                }
            }
        }
        __syncthreads();
        mask |= uint64_t(255) << shift;
        if (s_done) break;
    }
    // exactly rem keys of the bucket are >= the threshold
    const uint64_t thr = (uint64_t(bucket) << kHistBucketShift) | s_prefix;
    for (uint32_t i0 = 0; i0 < nb; i0 += kHistThreads) {
        const uint32_t i = i0 + t;
        const uint64_t k = i < nb ? src[i] : 0ull;
        const bool take = i < nb && k >= thr;
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        unsigned long long base = 0;
        if (lane == 0 && bal) base = atomicAdd((unsigned long long*)out_n, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) out[base + __popc(bal & ((1u << lane) - 1))] = k;
    }
}

// Keys above the boundary bucket go to out, the boundary bucket's keys to
// bkeys; the last CTA to finish (a ticket in SelectHist) resolves the bucket
// (resolve_bucket_cta) and re-zeroes the histogram for the next select — the
// compaction and the boundary resolution in one launch.
__global__ void __launch_bounds__(kHistThreads) hist_select_kernel(const uint64_t* __restrict__ keys,
                                                           const uint64_t* __restrict__ d_n, uint64_t want,
                                                           SelectHist* __restrict__ st, uint64_t* __restrict__ bkeys,
                                                           uint64_t* __restrict__ out, uint64_t* __restrict__ out_n,
                                                           const uint64_t* __restrict__ ukeys,
                                                           const uint64_t* __restrict__ d_nu) {
    dev::pdl_wait();
    const uint64_t n_all = *d_n;
    __shared__ HistBoundary hb;
    hist_boundary(st, n_all, want, hb);
    const bool all = hb.take_all;
    const uint32_t bucket = hb.bucket;
    // a boundary above the score-0 bucket selects positive scores only, and
    // every positive stage-2 score belongs to a candidate with a kept token:
    // scan that (much shorter) list when the producer kept one
    const bool use_u = ukeys && !all && bucket > kHistZeroBucket;
    if (use_u) keys = ukeys;
    const uint64_t n = use_u ? *d_nu : n_all;
    const uint32_t lane = threadIdx.x & 31;
    // one atomic per CTA and output (the CTA's warps take consecutive ranges):
    // per-warp atomics on the two counters queue on one L2 slice
    __shared__ uint32_t wa[32], wb[32];
    __shared__ unsigned long long ca, cb;
    const uint32_t warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (uint64_t b0 = uint64_t(blockIdx.x) * blockDim.x; b0 < n; b0 += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = b0 + threadIdx.x;
        const uint64_t k = i < n ? __ldcg(keys + i) : 0;
        const uint32_t b = uint32_t(k >> kHistBucketShift);
        const bool above = i < n && (all || b > bucket), inb = i < n && !all && b == bucket;
        const uint32_t ba = __ballot_sync(0xffffffffu, above), bb = __ballot_sync(0xffffffffu, inb);
        if (lane == 0) wa[warp] = __popc(ba), wb[warp] = __popc(bb);
        __syncthreads();
        if (threadIdx.x < 32) {
            // exclusive scans of the warp counts, one atomic per counter
            const uint32_t xa = lane < nwarps ? wa[lane] : 0u, xb = lane < nwarps ? wb[lane] : 0u;
            uint32_t ia = xa, ib = xb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
                if (lane >= uint32_t(o)) ia += ya, ib += yb;
            }
            const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
            if (lane == 0) {
                ca = ta ? atomicAdd((unsigned long long*)out_n, (unsigned long long)ta) : 0ull;
                cb = tb ? atomicAdd(&st->bn, (unsigned long long)tb) : 0ull;
            }
            if (lane < nwarps) wa[lane] = ia - xa, wb[lane] = ib - xb;
        }
        __syncthreads();
        if (above) out[ca + wa[warp] + __popc(ba & ((1u << lane) - 1))] = k;
        if (inb) bkeys[cb + wb[warp] + __popc(bb & ((1u << lane) - 1))] = k;
        __syncthreads();  // wa / wb / ca / cb are rewritten by the next round
    }
    // ---- the last CTA: boundary bucket, then a clean histogram
    __shared__ uint32_t s_last;
    if (threadIdx.x == 0) s_last = dev::last_ticket(&st->done, gridDim.x);
    __syncthreads();
    if (!s_last) return;
    const uint32_t nb = all ? 0u : uint32_t(__ldcg(&st->bn));
    if (nb) {
        if (nb <= kResolveStage) {
            extern __shared__ __align__(16) uint64_t sk[];
            for (uint32_t i = threadIdx.x; i < nb; i += kHistThreads) sk[i] = __ldcg(bkeys + i);
            __syncthreads();
            resolve_bucket_cta(sk, nb, hb.rem, bucket, out, out_n);
        } else {
            resolve_bucket_cta(bkeys, nb, hb.rem, bucket, out, out_n);
        }
    }
    // every CTA read the histogram before taking its ticket: clear the
    // non-empty blocks (their sums fetched in one round trip), then the sums
    // and the counters
    __shared__ uint32_t s_nz;
    if (threadIdx.x < 32) {
        const uint32_t nz = __ballot_sync(0xffffffffu, __ldcg(&st->blk[threadIdx.x]) != 0);
        if (threadIdx.x == 0) s_nz = nz;
        st->blk[threadIdx.x] = 0;
    }
    __syncthreads();
    for (uint32_t nz = s_nz; nz; nz &= nz - 1) {
        uint4* h4 = reinterpret_cast<uint4*>(st->hist + (__ffs(nz) - 1) * 2048);
        for (uint32_t i = threadIdx.x; i < 2048 / 4; i += kHistThreads) h4[i] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) st->bn = 0, st->done = 0;
}


// ---- global-exact shard exchange ---------------------------------------
// A key in GLOBAL form carries the global passage id: (score image << 32) |
// ~(local id + base).  Within one shard the map is monotone, so local and
// global forms order the shard's keys identically; across shards only the
// global form is comparable.
__device__ __forceinline__ uint64_t globalize(uint64_t key, uint32_t base) {
    return (key & 0xffffffff00000000ull) | uint64_t(~(dev::key_id(key) + base));
}

// out[j] = global form of keys[j] for j < min(*d_n, stride), 0 (below every
// real key) for the rest of the stride.
__global__ void export_keys_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                                   uint64_t stride, uint32_t base, uint64_t* __restrict__ out) {
    dev::pdl_wait();
    const uint64_t n = *d_n;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < stride;
         j += uint64_t(gridDim.x) * blockDim.x)
        out[j] = j < n ? globalize(keys[j], base) : 0ull;
}

// Exchange step of the single-process sharded searcher (engine.cpp,
// ShardedSearcher): row g of dst = `words` u64 of shard g's exported row,
// read straight from that shard's device memory through NVLink peer access
// (or locally when shards share a device) — the all-gather as one kernel.
__global__ void gather_rows_kernel(launch::PeerRows src, uint32_t shards, uint64_t words, uint64_t* __restrict__ dst) {
    dev::pdl_wait();
    const uint64_t total = uint64_t(shards) * words;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = e / words, j = e - g * words;
        dst[e] = __ldcv(src.p[g] + j);  // volatile: the peer wrote it this query
    }
}

// Per-query merge of shard top-k lists for a whole batch (throughput mode
// over passage shards): CTA j merges query j's lists — shard g's at
// pids/scores [g][B][k] with count counts[g][B] — into the global top-k by
// (score desc, pid asc) (pipeline.cpp:139-163): keys staged in shared memory,
// each key ranked against all (unique keys: rank = # greater).
constexpr uint32_t kMergeThreads = 256;
__global__ void __launch_bounds__(kMergeThreads)
merge_batch_kernel(const uint32_t* __restrict__ pids, const float* __restrict__ scores,
                   const uint64_t* __restrict__ counts, uint32_t shards, uint32_t B, uint32_t k,
                   uint32_t* __restrict__ out_pids, float* __restrict__ out_scores, uint64_t* __restrict__ out_n) {
    dev::pdl_wait();
    extern __shared__ uint64_t mk[];
    const uint32_t j = blockIdx.x;
    const uint32_t total = shards * k;
    for (uint32_t e = threadIdx.x; e < total; e += kMergeThreads) {
        const uint32_t g = e / k, r = e - g * k;
        const uint64_t off = (uint64_t(g) * B + j) * k + r;
        const uint64_t c = counts[uint64_t(g) * B + j];
        mk[e] = r < c ? dev::make_key(scores[off], pids[off]) : 0ull;
    }
    __syncthreads();
    uint32_t nz = 0;
    for (uint32_t e = threadIdx.x; e < total; e += kMergeThreads) {
        const uint64_t x = mk[e];
        if (!x) continue;
        ++nz;
        uint32_t rank = 0;
        for (uint32_t f = 0; f < total; ++f) rank += mk[f] > x;
        if (rank < k) {
            out_pids[uint64_t(j) * k + rank] = dev::key_id(x);
            out_scores[uint64_t(j) * k + rank] = dev::key_score(x);
        }
    }
    __shared__ uint32_t s_nz;
    if (threadIdx.x == 0) s_nz = 0;
    __syncthreads();
    atomicAdd(&s_nz, nz);
    __syncthreads();
    if (threadIdx.x == 0) out_n[j] = s_nz < k ? s_nz : k;
}

// One CTA.  (1) t = the want-th largest non-zero key of the gathered global
// keys g[0..total) by an MSB-first 8-bit radix select (t = 1, keep all, when
// fewer than `want` are non-zero); (2) keys[0..*d_n) (local form, this
// shard) keep exactly those whose global form is >= t, compacted in place in
// their original order; *d_n becomes the survivor count.  Because every
// shard's exported list holds its local top-`want`, the gathered union holds
// the global top-`want`, so the survivors are the global selection's members
// on this shard — the reference's single-index select_top (pipeline.cpp:139-163).
constexpr uint32_t kThrThreads = 1024;
__global__ void __launch_bounds__(kThrThreads)
threshold_filter_kernel(const uint64_t* __restrict__ g, uint64_t total, uint64_t want,
                        uint64_t* __restrict__ keys, uint64_t* __restrict__ d_n, uint32_t base) {
    dev::pdl_wait();
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix, s_rem;
    __shared__ uint32_t s_warp[kThrThreads / 32];
    __shared__ uint32_t s_out;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        s_prefix = 0;
        s_rem = want;
        s_out = 0;
    }
    // the first histogram pass also counts the non-zero gathered keys
    uint64_t prefix = 0;  // digits fixed so far (high bits), shifted into place
    bool keep_all = false;
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        for (uint32_t i = tid; i < 256; i += kThrThreads) hist[i] = 0;
        __syncthreads();
        const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (uint64_t i = tid; i < total; i += kThrThreads) {
            const uint64_t x = __ldcg(g + i);
            if (x != 0ull && (x & hi_mask) == prefix) atomicAdd(&hist[(x >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t rem = s_rem;
            if (pass == 0) {
                uint64_t nz = 0;
                for (int b = 0; b < 256; ++b) nz += hist[b];
                if (nz < want) rem = 0;  // keep all
            }
            if (rem == 0) {
                s_rem = 0;
            } else {
                int b = 255;
                for (; b > 0; --b) {
                    if (hist[b] >= rem) break;
                    rem -= hist[b];
                }
                s_prefix = prefix | (uint64_t(b) << shift);
                s_rem = rem;
            }
        }
        __syncthreads();
        if (s_rem == 0) {
            keep_all = true;
            break;
        }
        prefix = s_prefix;
    }
    const uint64_t t = keep_all ? 1ull : prefix;
    // (2) order-preserving in-place compaction, one 1024-key chunk at a time
    const uint64_t n = *d_n;
    const uint32_t lane = tid & 31u, warp = tid >> 5;
    for (uint64_t c0 = 0; c0 < n; c0 += kThrThreads) {
        const uint64_t i = c0 + tid;
        const uint64_t x = i < n ? keys[i] : 0ull;
        const bool ok = i < n && globalize(x, base) >= t;
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = 0;
        for (uint32_t w = 0; w < warp; ++w) before += s_warp[w];
        const uint32_t base_out = s_out;
        __syncthreads();
        if (ok) keys[base_out + before + __popc(bal & ((1u << lane) - 1u))] = x;
        if (tid == kThrThreads - 1) s_out = base_out + before + __popc(bal);
        __syncthreads();
    }
    if (tid == 0) *d_n = s_out;
}


// Top-`want` SET (unordered) of keys[0..*d_n), n <= kSmallSortMax, in one CTA:
// the keys are staged in shared memory, an MSB-first 8-bit radix select finds
// the want-th largest key t (keys are unique), and every key >= t is written
// to out (order unspecified; *d_out_n = min(n, want)).  Stage 3 needs only
// the set — stage 4 scores it and the final select orders the result.
constexpr uint32_t kSelCtaThreads = 1024;
__global__ void __launch_bounds__(kSelCtaThreads)
select_set_cta_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n, uint64_t want,
                      uint64_t* out, uint64_t* __restrict__ d_out_n, launch::FinalistScanArgs fs, uint32_t nmax) {
    dev::pdl_wait();
    // [keys | (with fs.cand_len) offsets, doclens, input index of each output]
    extern __shared__ uint64_t sk[];
    uint64_t* co = sk + nmax;
    uint32_t* cl = reinterpret_cast<uint32_t*>(co + nmax);
    uint32_t* sidx = cl + nmax;
    const bool carry = fs.pref && fs.cand_len;
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix, s_rem, s_mask;
    __shared__ uint32_t s_done, s_cnt;
    const uint32_t t = threadIdx.x;
    const uint32_t n = uint32_t(*d_n);
    for (uint32_t i = t; i < n; i += kSelCtaThreads) {
        sk[i] = __ldcg(keys + i);
        if (carry) co[i] = __ldcg(fs.cand_off + i), cl[i] = __ldcg(fs.cand_len + i);
    }
    if (t == 0) {
        s_prefix = 0, s_rem = want, s_mask = 0, s_done = n <= want, s_cnt = 0;
    }
    __syncthreads();
    if (s_done) {  // everything survives
        for (uint32_t i = t; i < n; i += kSelCtaThreads) {
            out[i] = sk[i];
            if (carry) sidx[i] = i;
        }
        if (t == 0) *d_out_n = n;
        if (fs.pref) {
            __syncthreads();
            if (carry) fused::finalist_scan_carried(n, sidx, cl, co, fs.pref, fs.fin_base, fs.tokens, fs.run_p0);
            else fused::finalist_scan(nullptr, out, n, fs.doclens, fs.offsets, fs.pref, fs.fin_base, fs.tokens, fs.run_p0);
        }
        return;
    }
    for (int shift = 56; shift >= 0 && !s_done; shift -= 8) {
        for (uint32_t b = t; b < 256; b += kSelCtaThreads) hist[b] = 0;
        __syncthreads();
        const uint64_t mask = s_mask, prefix = s_prefix;
        for (uint32_t i = t; i < n; i += kSelCtaThreads)
            if ((sk[i] & mask) == prefix) atomicAdd(&hist[(sk[i] >> shift) & 255u], 1u);
        __syncthreads();
        if (t < 32) {
            // bins 255 - 8 t .. 248 - 8 t per lane (lane 0 the highest), prefix from the top
            uint32_t c[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) sum += (c[j] = hist[255 - 8 * t - j]);
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (t >= uint32_t(o)) incl += y;
            }
            const uint64_t rem = s_rem;
            uint64_t above = incl - sum;
            if (above < rem && rem <= above + sum) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (above < rem && rem <= above + c[j]) {
                        const uint32_t b = 255 - 8 * t - j;
                        s_prefix = prefix | (uint64_t(b) << shift);
                        s_mask = mask | (uint64_t(255) << shift);
                        s_rem = rem - above;
                        s_done = c[j] == rem - above;  // the whole bucket is taken
                    }
                    above += c[j];
                }
            }
        }
        __syncthreads();
    }
    // the threshold: the bucket prefix when the whole bucket is taken, else
    // the fully resolved key (64 bits of prefix) — keys >= it survive
    const uint64_t thr = s_prefix;
    for (uint32_t i0 = 0; i0 < n; i0 += kSelCtaThreads) {
        const uint32_t i = i0 + t;
        const bool ok = i < n && sk[i] >= thr;
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        uint32_t base = 0;
        if ((t & 31) == 0 && bal) base = atomicAdd(&s_cnt, uint32_t(__popc(bal)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (ok) {
            const uint32_t pos = base + __popc(bal & ((1u << (t & 31)) - 1u));
            out[pos] = sk[i];
            if (carry) sidx[pos] = i;
        }
    }
    if (t == 0) *d_out_n = want;
    if (fs.pref) {  // stage 4's finalist scan over the set just written, same CTA
        __syncthreads();
        if (carry)
            fused::finalist_scan_carried(uint32_t(want), sidx, cl, co, fs.pref, fs.fin_base, fs.tokens, fs.run_p0);
        else
            fused::finalist_scan(nullptr, out, uint32_t(want), fs.doclens, fs.offsets, fs.pref, fs.fin_base,
                                 fs.tokens, fs.run_p0);
    }
}

}  // namespace

namespace launch {

void select_top_hist(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want, SelectHist* d_st,
                     uint64_t* d_bkeys, uint64_t* d_out_keys, uint64_t* d_out_n, cudaStream_t st,
                     const uint64_t* d_ukeys, const uint64_t* d_nu) {
    if (nmax == 0) return;
    // one 1024-thread CTA per SM at most; the last one stages the boundary bucket
    const uint32_t grid = grid_for(nmax, kHistThreads, uint32_t(sm_count()));
    static launch::PerDeviceOnce cfg;
    if (cfg.first())
        cudaFuncSetAttribute(hist_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kResolveStage * sizeof(uint64_t)));
    ::plaid::launch::pdl(hist_select_kernel, grid, kHistThreads, kResolveStage * sizeof(uint64_t), st, d_keys, d_n, want, d_st, d_bkeys, d_out_keys,
                         d_out_n, d_ukeys, d_nu);
    count_launch();
}

void select_top_large(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want,
                      SelectState* d_state, uint64_t* d_out_keys, uint64_t* d_out_n,
                      cudaStream_t st) {
    // state (histograms, barrier counter) and the output count start at zero
    cudaMemsetAsync(d_state, 0, kSelectStateZeroBytes, st);
    cudaMemsetAsync(d_out_n, 0, sizeof(uint64_t), st);
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, radix_select_kernel, kSelThreads, 0);
        if (per_sm < 1) per_sm = 1;
        if (per_sm > 2) per_sm = 2;
    }
    const uint32_t grid = grid_for(nmax, kSelThreads * 4, uint32_t(sm_count() * per_sm));
    void* args[] = {(void*)&d_keys, (void*)&d_n, (void*)&want, (void*)&d_state, (void*)&d_out_keys,
                    (void*)&d_out_n};
    cudaLaunchCooperativeKernel((const void*)radix_select_kernel, dim3(grid), dim3(kSelThreads), args, 0, st);
    count_launch();
}

uint64_t sort_tmp_capacity(uint64_t nmax) { return nmax <= kSmallSortMax ? 0 : next_pow2(nmax); }

void finalize_rank(const uint32_t* d_ids, const uint64_t* d_fkeys, const uint64_t* d_n, uint64_t nmax, uint32_t rows,
                   uint32_t* d_run, uint64_t want, uint32_t* d_out_ids, float* d_out_scores, uint64_t* d_out_n,
                   uint32_t id_base, unsigned int* d_ticket, cudaStream_t st) {
    if (nmax < kFinalRankMin || nmax > kSmallSortMax) fail_cuda_driver(1, "finalize_rank: nmax out of range");
    // one 32 x 33 float tile per warp, then the nmax keys
    const size_t smem = kFinTileWords * sizeof(float) + size_t(nmax) * sizeof(uint64_t);
    static launch::PerDeviceOnce cfg;
    if (cfg.first())
        cudaFuncSetAttribute(finalize_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kFinTileWords * sizeof(float) + kSmallSortMax * sizeof(uint64_t)));
    const uint32_t grid = uint32_t((nmax + kFinRankPerCta - 1) / kFinRankPerCta);
    ::plaid::launch::pdl(finalize_rank_kernel, grid, kFinRankThreads, smem, st, d_ids, d_fkeys, d_n, rows, d_run, want,
                         d_out_ids, d_out_scores, d_out_n, id_base, d_ticket);
    count_launch();
}

void sort_top(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want,
              uint64_t* d_out_keys, uint32_t* d_out_ids, float* d_out_scores, uint64_t* d_out_n,
              uint32_t id_base, uint64_t* d_tmp, cudaStream_t st) {
    if (nmax <= kSmallSortMax && nmax >= 256) {
        const size_t smem = size_t(4) * (rank_quarter_pairs(uint32_t(nmax)) + 1) * 16;
        static launch::PerDeviceOnce rank_cfg;
        if (rank_cfg.first()) {
            cudaFuncSetAttribute(sort_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(4 * (rank_quarter_pairs(uint32_t(kSmallSortMax)) + 1) * 16));
        }
        const uint32_t grid = uint32_t((nmax + kRankPerCta - 1) / kRankPerCta);
        ::plaid::launch::pdl(sort_rank_kernel, grid, kRankThreads, smem, st, d_keys, d_n, want, d_out_keys, d_out_ids, d_out_scores,
                                                          d_out_n, id_base);
        count_launch();
        return;
    }
    if (nmax <= kSmallSortMax) {
        const uint32_t npad = uint32_t(next_pow2(nmax < 2 ? 2 : nmax));
        const size_t smem = size_t(npad) * sizeof(uint64_t);
        static launch::PerDeviceOnce configured;
        if (configured.first()) {
            cudaFuncSetAttribute(sort_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kSmallSortMax * sizeof(uint64_t)));
        }
        const uint32_t threads = npad / 2 < 1024 ? (npad / 2 < 32 ? 32 : npad / 2) : 1024;
        ::plaid::launch::pdl(sort_small_kernel, 1, threads, smem, st, d_keys, d_n, npad, want, d_out_keys, d_out_ids,
                                                    d_out_scores, d_out_n, id_base);
        count_launch();
        return;
    }
    const uint64_t npad = next_pow2(nmax);
    const uint32_t grid = grid_for(npad, 256, uint32_t(sm_count()) * 8);
    ::plaid::launch::pdl(pad_copy_kernel, grid, 256, 0, st, d_keys, d_n, npad, d_tmp);
    count_launch();
    for (uint64_t k = 2; k <= npad; k <<= 1)
        for (uint64_t j = k >> 1; j > 0; j >>= 1) {
            ::plaid::launch::pdl(bitonic_step_kernel, grid, 256, 0, st, d_tmp, npad, j, k);
            count_launch();
        }
    ::plaid::launch::pdl(emit_kernel, grid_for(want, 256, 4096), 256, 0, st, d_tmp, d_n, want, d_out_keys, d_out_ids,
                                                          d_out_scores, d_out_n, id_base);
    count_launch();
}

void make_keys(const uint32_t* d_ids, const float* d_scores, uint64_t n, uint64_t* d_keys,
               cudaStream_t st) {
    ::plaid::launch::pdl(make_keys_kernel, grid_for(n, 256, 4096), 256, 0, st, d_ids, d_scores, n, d_keys);
    count_launch();
}

void merge_topk(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts,
                uint64_t shards, uint64_t stride, uint64_t count_stride, uint64_t per, uint64_t k,
                uint64_t* d_tmp_keys, uint64_t* d_tmp_n, uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n,
                uint64_t* d_sort_tmp, cudaStream_t st) {
    ::plaid::launch::pdl(merge_keys_kernel, grid_for(shards * per, 256, 4096), 256, 0, st,
        d_pids, d_scores, d_counts, shards, stride, count_stride, per, d_tmp_keys, d_tmp_n);
    count_launch();
    sort_top(d_tmp_keys, d_tmp_n, shards * per, k, nullptr, d_out_pids, d_out_scores, d_out_n, 0,
             d_sort_tmp, st);
}

void copy_count(const uint64_t* src, uint64_t* dst, uint64_t cap, cudaStream_t st) {
    ::plaid::launch::pdl(copy_count_kernel, 1, 1, 0, st, src, dst, cap);
    count_launch();
}

// Results of the host path straight into the caller's pinned (mapped)
// buffer, then a sequence flag (the host spins on it instead of a stream
// synchronize): one CTA after the final select.
__global__ void __launch_bounds__(256) publish_kernel(const uint4* __restrict__ src, uint4* dst, uint64_t n16,
                                                      unsigned int* dev_seq, volatile unsigned int* host_flag) {
    dev::pdl_wait();
    for (uint64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int seq = *dev_seq + 1;
        *dev_seq = seq;
        __threadfence_system();
        *host_flag = seq;
    }
}

void query_prologue(const float* d_q, uint32_t rows, uint32_t dim, int* d_status, uint32_t* d_zero, uint64_t nwords,
                    uint32_t* d_zero2, uint64_t nwords2, cudaStream_t st, const float* d_qsrc, void* d_qimg,
                    float* d_qcopy) {
    const uint64_t n16 = nwords / 4, m16 = nwords2 / 4;  // both regions are multiples of 16 bytes
    const bool img = d_qimg && d_qsrc && dim == 128 && rows <= 32;
    // at least one thread per query-image granule (the rows may be in host memory)
    // + one CTA for the norm check when validating
    const uint32_t grid = grid_for(std::max<uint64_t>(n16 + m16, img ? kQImgBytes / 16 : 0), 256,
                                   uint32_t(sm_count())) + (d_q ? 1u : 0u);
    static launch::PerDeviceOnce cfg;
    if (cfg.first())  // keep the SMs' shared-memory partition at its maximum so the
                      // S_cq CTAs (213 KB each) can become resident beside this grid
        cudaFuncSetAttribute(query_prologue_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    ::plaid::launch::pdl(query_prologue_kernel, grid, 256, 0, st, d_q, rows, dim, d_status,
                         reinterpret_cast<uint4*>(d_zero), n16, reinterpret_cast<uint4*>(d_zero2), m16,
                         (img || d_qcopy) ? d_qsrc : nullptr, img ? reinterpret_cast<uint4*>(d_qimg) : nullptr,
                         d_qcopy, d_qcopy ? rows * dim / 4 : 0u);
    count_launch();
}

void publish(const uint32_t* d_src, uint32_t* h_dst_mapped, uint64_t words, unsigned int* d_seq,
             unsigned int* h_flag_mapped, cudaStream_t st) {
    ::plaid::launch::pdl(publish_kernel, 1, 256, 0, st, reinterpret_cast<const uint4*>(d_src),
                         reinterpret_cast<uint4*>(h_dst_mapped), (words + 3) / 4, d_seq, h_flag_mapped);
    count_launch();
}

bool pdl_enabled() {
    static const bool on = getenv("PLAID_NO_PDL") == nullptr;
    return on;
}

void export_keys(const uint64_t* d_keys, const uint64_t* d_n, uint64_t stride, uint32_t base, uint64_t* d_out,
                 cudaStream_t st) {
    if (!stride) return;
    ::plaid::launch::pdl(export_keys_kernel, grid_for(stride, 256, 1024), 256, 0, st, d_keys, d_n, stride, base, d_out);
    count_launch();
}

void gather_rows(const PeerRows& src, uint32_t shards, uint64_t words, uint64_t* d_dst, cudaStream_t st) {
    if (!words || !shards) return;
    ::plaid::launch::pdl(gather_rows_kernel, grid_for(uint64_t(shards) * words, 256, 1024), 256, 0, st, src, shards,
                         words, d_dst);
    count_launch();
}

void merge_batch(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts, uint32_t shards, uint32_t B,
                 uint32_t k, uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n, cudaStream_t st) {
    if (!B) return;
    const size_t smem = size_t(shards) * k * sizeof(uint64_t);
    static launch::PerDeviceOnce cfg;
    if (cfg.first())
        cudaFuncSetAttribute(merge_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    ::plaid::launch::pdl(merge_batch_kernel, B, kMergeThreads, smem, st, d_pids, d_scores, d_counts, shards, B, k,
                         d_out_pids, d_out_scores, d_out_n);
    count_launch();
}

void threshold_filter(const uint64_t* d_gathered, uint64_t total, uint64_t want, uint64_t* d_keys, uint64_t* d_n,
                      uint32_t base, cudaStream_t st) {
    ::plaid::launch::pdl(threshold_filter_kernel, 1, kThrThreads, 0, st, d_gathered, total, want, d_keys, d_n, base);
    count_launch();
}

void select_set(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want, uint64_t* d_out_keys,
                uint64_t* d_out_n, const FinalistScanArgs* fs, cudaStream_t st) {
    const uint64_t nm = std::max<uint64_t>(nmax, 1);
    // keys, then (carried scan inputs) offsets, doclens and the output -> input map
    const bool carry = fs && fs->pref && fs->cand_len;
    const size_t smem = nm * (carry ? 24 : 8);
    static launch::PerDeviceOnce cfg;
    if (cfg.first()) {
        cudaFuncSetAttribute(select_set_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kSmallSortMax * 24));
    }
    ::plaid::launch::pdl(select_set_cta_kernel, 1, kSelCtaThreads, smem, st, d_keys, d_n, want, d_out_keys, d_out_n,
                         fs ? *fs : FinalistScanArgs{}, uint32_t(nm));
    count_launch();
}

}  // namespace launch
}  // namespace plaid
