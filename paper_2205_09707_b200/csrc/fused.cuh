// fused.cuh — CTA-level bodies shared by more than one kernel, so that a
// latency-bound step can ride inside the launch of its neighbour instead of
// paying its own kernel boundary (~2.8 us each in the PDL chain, measured by
// tools/pdl_chain.cu).  Device-only; included by .cu files.
#pragma once

#include <cstdint>

#include "device.cuh"

namespace plaid {
namespace fused {

// Kept-centroid list (interaction.cu, stage 2): blocks blk of nblk over the
// keep bitmap; list[] = kept centroid ids (order unspecified), counts[0] =
// number kept, counts[1] = total length of their posting lists.
__device__ __forceinline__ void keep_list(uint32_t blk, uint32_t nblk, const uint32_t* __restrict__ keep_bits,
                                          uint64_t K, const uint64_t* __restrict__ ivf_offsets,
                                          uint32_t* __restrict__ list, unsigned long long* __restrict__ counts) {
    const uint32_t lane = dev::lane_id();
    const uint64_t words = (K + 31) / 32;
    for (uint64_t w0 = (uint64_t(blk) * blockDim.x + threadIdx.x) & ~31ull; w0 < words;
         w0 += uint64_t(nblk) * blockDim.x) {
        const uint64_t w = w0 + lane;
        uint32_t bits = w < words ? keep_bits[w] : 0u;
        if (w == words - 1 && (K & 31)) bits &= (1u << (K & 31)) - 1;
        const uint32_t cnt = __popc(bits);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        if (!tot) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(counts, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        uint32_t slot = uint32_t(base) + incl - cnt;
        unsigned long long post = 0;
        while (bits) {
            const uint32_t c = uint32_t(w * 32 + (__ffs(bits) - 1));
            bits &= bits - 1;
            list[slot++] = c;
            post += ivf_offsets[c + 1] - ivf_offsets[c];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) post += __shfl_xor_sync(0xffffffffu, post, o);
        if (lane == 0) atomicAdd(counts + 1, post);
    }
}

// Stage-4 finalist scan (rank128.cu), one CTA of exactly 1024 threads:
// pref[p] = exclusive prefix of the finalists' doclens, fin_base[p] =
// offsets[pid] - pref[p], pref[n] = total (also *tokens when given), and
// (run_p0 given) run_p0[r] = the finalist holding stream position 32 r, so a
// warp of the tensor-core stage 4 finds the finalists of its 32-token run
// with one load.  The finalist pid is ids[p] or the id of keys[p].
__device__ __forceinline__ void finalist_scan(const uint32_t* __restrict__ ids, const uint64_t* keys, uint32_t n,
                                              const uint32_t* __restrict__ doclens,
                                              const uint64_t* __restrict__ offsets, uint32_t* __restrict__ pref,
                                              uint64_t* __restrict__ fin_base, uint64_t* __restrict__ tokens,
                                              uint32_t* __restrict__ run_p0 = nullptr) {
    __shared__ uint32_t warp_sums[32];
    auto pid_of = [&](uint32_t p) { return ids ? ids[p] : dev::key_id(keys[p]); };
    const uint32_t per = (n + 1023) / 1024;
    const uint32_t b = threadIdx.x * per, e = b + per < n ? b + per : n;
    uint32_t local = 0;
    for (uint32_t p = b; p < e; ++p) local += doclens[pid_of(p)];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = warp_sums[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= uint32_t(o)) wi += y;
        }
        warp_sums[lane] = wi - w;  // exclusive
    }
    __syncthreads();
    uint32_t run = warp_sums[warp] + incl - local;
    for (uint32_t p = b; p < e; ++p) {
        const uint32_t pid = pid_of(p);
        pref[p] = run;
        fin_base[p] = offsets[pid] - run;  // index token = fin_base[p] + stream position
        const uint32_t len = doclens[pid];
        if (run_p0)
            for (uint32_t r = (run + 31) / 32; 32 * r < run + len; ++r) run_p0[r] = p;
        run += len;
    }
    if (threadIdx.x == 1023) {
        pref[n] = warp_sums[31] + incl;  // total (last thread's inclusive)
        if (tokens) *tokens = pref[n];
    }
}

// finalist_scan with each finalist's (doclen, offset) already in shared
// memory: finalist p is select input idx[p], whose doclen / offset are
// len[idx[p]] / off[idx[p]] (carried from the stage-3 scorer).
__device__ __forceinline__ void finalist_scan_carried(uint32_t n, const uint32_t* idx, const uint32_t* len,
                                                      const uint64_t* off, uint32_t* __restrict__ pref,
                                                      uint64_t* __restrict__ fin_base, uint64_t* __restrict__ tokens,
                                                      uint32_t* __restrict__ run_p0) {
    __shared__ uint32_t warp_sums[32];
    const uint32_t per = (n + 1023) / 1024;
    const uint32_t b = threadIdx.x * per, e = b + per < n ? b + per : n;
    uint32_t local = 0;
    for (uint32_t p = b; p < e; ++p) local += len[idx[p]];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = warp_sums[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= uint32_t(o)) wi += y;
        }
        warp_sums[lane] = wi - w;  // exclusive
    }
    __syncthreads();
    uint32_t run = warp_sums[warp] + incl - local;
    for (uint32_t p = b; p < e; ++p) {
        const uint32_t i = idx[p], l = len[i];
        pref[p] = run;
        fin_base[p] = off[i] - run;  // index token = fin_base[p] + stream position
        if (run_p0)
            for (uint32_t r = (run + 31) / 32; 32 * r < run + l; ++r) run_p0[r] = p;
        run += l;
    }
    if (threadIdx.x == 1023) {
        pref[n] = warp_sums[31] + incl;  // total (last thread's inclusive)
        if (tokens) *tokens = pref[n];
    }
}

}  // namespace fused
}  // namespace plaid
