// candidates.cu — stage-1 candidate generation (pipeline.cpp:52-87).
//
// The union of the probed centroids' postings is formed in an N-bit bitmap
// (atomicOr per posting; duplicates across query tokens collapse for free),
// then compacted into ascending passage ids.  Scanning the bitmap in order is
// exactly the reference's `std::sort` of the unique ids (pipeline.cpp:83), so
// the output is bit-identical.  The search path compacts in one pass
// (decoupled look-back over published chunk counts); the standalone entry
// point uses two launches (per-chunk popcounts, then the writes).
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr uint32_t kChunkWords = 2048;  // 65536 passages per chunk
constexpr uint32_t kThreads = 256;
constexpr uint32_t kWordsPerThread = kChunkWords / kThreads;

__global__ void postings_bitmap_kernel(const uint64_t* __restrict__ ivf_offsets,
                                       const uint32_t* __restrict__ postings,
                                       const uint32_t* __restrict__ sel,
                                       uint32_t* __restrict__ bitmap) {
    dev::pdl_wait();
    const uint32_t c = sel[blockIdx.x];
    const uint64_t b = ivf_offsets[c], e = ivf_offsets[c + 1];
    for (uint64_t j = b + threadIdx.x; j < e; j += blockDim.x) {
        const uint32_t p = postings[j];
        atomicOr(bitmap + (p >> 5), 1u << (p & 31));
    }
}

__device__ __forceinline__ uint32_t masked_word(const uint32_t* bitmap, uint64_t w, uint64_t N) {
    const uint64_t words = (N + 31) / 32;
    if (w >= words) return 0;
    uint32_t v = bitmap[w];
    if (w == words - 1 && (N & 31)) v &= (1u << (N & 31)) - 1;
    return v;
}

__global__ void chunk_count_kernel(const uint32_t* __restrict__ bitmap, uint64_t N,
                                   uint32_t* __restrict__ counts) {
    dev::pdl_wait();
    __shared__ uint32_t warp_sums[kThreads / 32];
    const uint64_t w0 = uint64_t(blockIdx.x) * kChunkWords + threadIdx.x * kWordsPerThread;
    uint32_t n = 0;
#pragma unroll
    for (uint32_t j = 0; j < kWordsPerThread; ++j) n += __popc(masked_word(bitmap, w0 + j, N));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t k = 0; k < kThreads / 32; ++k) t += warp_sums[k];
        counts[blockIdx.x] = t;
    }
}

__global__ void chunk_write_kernel(const uint32_t* __restrict__ bitmap, uint64_t N,
                                   const uint32_t* __restrict__ counts, uint32_t* __restrict__ out,
                                   uint64_t* __restrict__ out_n, uint32_t* __restrict__ slot_of) {
    dev::pdl_wait();
    __shared__ uint64_t red[kThreads / 32];
    __shared__ uint32_t scan[kThreads / 32];
    // base = sum of counts of the chunks before this one
    uint64_t part = 0;
    for (uint32_t c = threadIdx.x; c < blockIdx.x; c += kThreads) part += counts[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;

    const uint64_t w0 = uint64_t(blockIdx.x) * kChunkWords + threadIdx.x * kWordsPerThread;
    uint32_t words[kWordsPerThread];
    uint32_t mine = 0;
#pragma unroll
    for (uint32_t j = 0; j < kWordsPerThread; ++j) {
        words[j] = masked_word(bitmap, w0 + j, N);
        mine += __popc(words[j]);
    }
    // block exclusive scan of `mine`
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += v;
    }
    if (lane == 31) scan[warp] = incl;
    __syncthreads();
    uint64_t base = 0;
    for (uint32_t k = 0; k < kThreads / 32; ++k) base += red[k];
    uint32_t before = 0;
    for (uint32_t k = 0; k < warp; ++k) before += scan[k];
    uint64_t pos = base + before + incl - mine;
#pragma unroll
    for (uint32_t j = 0; j < kWordsPerThread; ++j) {
        uint32_t v = words[j];
        while (v) {
            const uint32_t b = __ffs(v) - 1;
            v &= v - 1;
            const uint32_t pid = uint32_t((w0 + j) * 32 + b);
            if (slot_of) slot_of[pid] = uint32_t(pos);
            out[pos++] = pid;
        }
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kThreads - 1) *out_n = pos;
}


// Single pass (decoupled look-back): every chunk publishes its popcount with
// a ready flag, then sums its predecessors' published counts (spinning on
// their flags) and writes its ids in order.  A CTA takes its chunk from a
// ticket counter (status[nchunks]), not from blockIdx.x: CTAs are not
// dispatched in blockIdx order, and with more chunks than resident CTAs a
// CTA spinning on a lower chunk that was never scheduled would deadlock.
// With tickets every lower chunk belongs to a CTA that is already running.
// `status` (nchunks + 1 u64) must be zero on entry (the per-query prologue
// clears it).
__global__ void chunk_compact_kernel(const uint32_t* __restrict__ bitmap, uint64_t N,
                                     unsigned long long* __restrict__ status, uint32_t* __restrict__ out,
                                     uint64_t* __restrict__ out_n, uint32_t* __restrict__ slot_of) {
    dev::pdl_wait();
    __shared__ uint64_t red[kThreads / 32];
    __shared__ uint32_t scan[kThreads / 32];
    __shared__ uint32_t ticket;
    constexpr unsigned long long kReady = 1ull << 63;
    if (threadIdx.x == 0) ticket = uint32_t(atomicAdd(status + gridDim.x, 1ull));
    __syncthreads();
    const uint32_t chunk = ticket;
    const uint64_t w0 = uint64_t(chunk) * kChunkWords + threadIdx.x * kWordsPerThread;
    uint32_t words[kWordsPerThread];
    uint32_t mine = 0;
#pragma unroll
    for (uint32_t j = 0; j < kWordsPerThread; ++j) {
        words[j] = masked_word(bitmap, w0 + j, N);
        mine += __popc(words[j]);
    }
    // block inclusive scan of `mine`
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += v;
    }
    if (lane == 31) scan[warp] = incl;
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (uint32_t k = 0; k < kThreads / 32; ++k) {
        if (k < warp) before += scan[k];
        total += scan[k];
    }
    if (threadIdx.x == 0) {
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(status + chunk), "l"(kReady | total) : "memory");
    }
    // look back: the counts of every earlier chunk
    uint64_t part = 0;
    for (uint32_t c = threadIdx.x; c < chunk; c += kThreads) {
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(status + c) : "memory");
        } while (!(v & kReady));
        part += v & ~kReady;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    uint64_t base = 0;
    for (uint32_t k = 0; k < kThreads / 32; ++k) base += red[k];
    uint64_t pos = base + before + incl - mine;
#pragma unroll
    for (uint32_t j = 0; j < kWordsPerThread; ++j) {
        uint32_t v = words[j];
        while (v) {
            const uint32_t b = __ffs(v) - 1;
            v &= v - 1;
            const uint32_t pid = uint32_t((w0 + j) * 32 + b);
            if (slot_of) slot_of[pid] = uint32_t(pos);
            out[pos++] = pid;
        }
    }
    if (chunk == gridDim.x - 1 && threadIdx.x == kThreads - 1) *out_n = pos;
}

}  // namespace

namespace launch {

void postings_to_bitmap(const IndexView& ix, const uint32_t* d_sel, uint32_t nsel,
                        uint32_t* d_bitmap, cudaStream_t st) {
    if (nsel == 0) return;
    ::plaid::launch::pdl(postings_bitmap_kernel, nsel, 256, 0, st, ix.ivf_offsets, ix.ivf_postings, d_sel, d_bitmap);
    count_launch();
}

uint32_t bitmap_chunks(uint64_t N) {
    const uint64_t words = (N + 31) / 32;
    uint64_t c = (words + kChunkWords - 1) / kChunkWords;
    return uint32_t(c ? c : 1);
}

void bitmap_compact_1pass(const uint32_t* d_bitmap, uint64_t N, unsigned long long* d_status, uint32_t* d_out_ids,
                          uint64_t* d_out_n, uint32_t* d_slot_of, cudaStream_t st) {
    ::plaid::launch::pdl(chunk_compact_kernel, bitmap_chunks(N), kThreads, 0, st, d_bitmap, N, d_status, d_out_ids,
                         d_out_n, d_slot_of);
    count_launch();
}

void bitmap_compact(const uint32_t* d_bitmap, uint64_t N, uint32_t* d_chunk_counts,
                    uint32_t* d_out_ids, uint64_t* d_out_n, uint32_t* d_slot_of, cudaStream_t st) {
    const uint32_t chunks = bitmap_chunks(N);
    ::plaid::launch::pdl(chunk_count_kernel, chunks, kThreads, 0, st, d_bitmap, N, d_chunk_counts);
    ::plaid::launch::pdl(chunk_write_kernel, chunks, kThreads, 0, st, d_bitmap, N, d_chunk_counts, d_out_ids, d_out_n,
                         d_slot_of);
    count_launch();
    count_launch();
}

}  // namespace launch
}  // namespace plaid
