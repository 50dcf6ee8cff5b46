// interaction.cu — centroid interaction, stages 2 and 3 (pipeline.cpp:97-137).
//
// Per candidate passage: acc[j] = max over its (unmasked) tokens t of
// S[code(t)][j]; score = in-order fp32 sum of acc[0..|Q|) if any row was used,
// else exactly 0.  The max is order-independent except for the sign of zero,
// and an in-order sum that starts from +0.0f is insensitive to that sign, so
// the scores are bit-identical to the reference.
//
// Stage 2 (masked, candidate count up to N): padding-free flattened scan.  A
// block takes 256 candidates, prefix-sums their doclens in shared memory and
// lets its 256 threads sweep the concatenated token range, so consecutive
// threads read consecutive codes regardless of passage boundaries.  Tokens on
// kept centroids (few) are queued in shared memory and then folded warp-wide:
// one 128-byte S row per entry, atomicMax on an order-preserving integer image
// of the accumulator.  Stage 3 (unmasked, <= ndocs candidates): one warp per
// passage, codes broadcast by shuffle, 8 S-row loads in flight per warp.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "fused.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr uint32_t kCB = 256;         // candidates per block (stage 2)
constexpr uint32_t kListCap = 1024;   // kept-token queue per block (static smem < 48 KB)
constexpr uint32_t kAccPitch = 33;    // conflict-free column sums
constexpr uint64_t kListsPerCandidate = 4;  // kept postings per C1 candidate above which ci_all runs

__device__ __forceinline__ uint32_t cand_id(const uint32_t* ids, const uint64_t* keys, uint64_t i) {
    return ids ? ids[i] : dev::key_id(keys[i]);
}

__device__ __forceinline__ bool kept(const uint32_t* keep_bits, uint32_t code) {
    return (__ldg(keep_bits + (code >> 5)) >> (code & 31)) & 1u;
}

// Warp-wide scoring of one passage (also the overflow fallback of stage 2).
// Returns the score on every lane; *used = rows folded in.
template <bool MASKED>
__device__ float score_passage_warp(const uint32_t* __restrict__ codes, uint64_t off, uint32_t len,
                                    const float* __restrict__ S, uint32_t rows,
                                    const uint32_t* __restrict__ keep_bits, uint32_t* used_out) {
    const uint32_t lane = dev::lane_id();
    float acc = -INFINITY;
    uint32_t used = 0;
    for (uint32_t base = 0; base < len; base += 32) {
        const uint32_t t = base + lane;
        const uint32_t code = t < len ? __ldg(codes + off + t) : 0u;
        bool valid = t < len;
        if (MASKED) valid = valid && kept(keep_bits, code);
        uint32_t bits = __ballot_sync(0xffffffffu, valid);
        used += __popc(bits);
        if (!bits) continue;  // every token of the chunk masked
        // all 32 S-row gathers of the chunk in flight at once, then the
        // maxima in token order (`if (s > acc)`, pipeline.cpp:121-123).  The
        // loads are unpredicated (a predicated load holds one of the 7
        // predicate registers until it lands, capping the loads in flight):
        // slots past the chunk's valid tokens repeat the last valid one,
        // which cannot change a strict running max
        const int last = 31 - __clz(bits);
        float s[32];
#pragma unroll
        for (int v = 0; v < 32; ++v) {
            const int b = bits ? __ffs(bits) - 1 : last;
            const uint32_t c = __shfl_sync(0xffffffffu, code, b);
            s[v] = __ldg(S + uint64_t(c) * kScoresPitch + lane);
            bits &= bits - 1;
        }
#pragma unroll
        for (int v = 0; v < 32; ++v) acc = dev::max_gt(acc, s[v]);
    }
    float total = 0.0f;
    if (used > 0) {
        for (uint32_t j = 0; j < rows; ++j) total = __fadd_rn(total, __shfl_sync(0xffffffffu, acc, j));
    }
    *used_out = used;
    return total;
}

// Stage 3 (and the unmasked entry point): one warp per passage.
__global__ void __launch_bounds__(256)
ci_warp_kernel(const uint32_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
               const uint32_t* __restrict__ doclens, const float* __restrict__ S, uint32_t rows,
               const uint32_t* __restrict__ ids, const uint64_t* __restrict__ keys,
               const uint64_t* __restrict__ d_n, const uint32_t* __restrict__ keep_bits,
               uint64_t* __restrict__ out_keys, float* __restrict__ out_scores,
               unsigned long long* __restrict__ d_rows, uint32_t* __restrict__ out_len,
               uint64_t* __restrict__ out_off) {
    dev::pdl_wait();
    const uint64_t n = *d_n;
    const uint32_t lane = dev::lane_id();
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    unsigned long long rows_local = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const uint32_t pid = cand_id(ids, keys, i);
        const uint64_t off = offsets[pid];
        const uint32_t len = doclens[pid];
        uint32_t used;
        float total = keep_bits ? score_passage_warp<true>(codes, off, len, S, rows, keep_bits, &used)
                                : score_passage_warp<false>(codes, off, len, S, rows, keep_bits, &used);
        if (lane == 0) {
            out_keys[i] = dev::make_key(total, pid);
            if (out_scores) out_scores[i] = total;
            if (out_len) out_len[i] = len, out_off[i] = off;
        }
        rows_local += used;
    }
    dev::block_add_lane0(d_rows, rows_local);
}

// Stage 2: masked, flattened over the block's concatenated token range.
__global__ void __launch_bounds__(kCB)
ci_masked_flat_kernel(const uint32_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                      const uint32_t* __restrict__ doclens, const float* __restrict__ S,
                      uint32_t rows, const uint32_t* __restrict__ ids,
                      const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                      const uint32_t* __restrict__ keep_bits, const uint32_t* __restrict__ owners,
                      uint64_t* __restrict__ out_keys, float* __restrict__ out_scores,
                      unsigned long long* __restrict__ d_rows) {
    dev::pdl_wait();
    __shared__ uint64_t off_s[kCB];
    __shared__ uint32_t start_s[kCB + 1];
    __shared__ uint32_t acc_s[kCB * kAccPitch];
    __shared__ uint32_t used_s[kCB];
    __shared__ uint32_t list_s[kListCap * 2];
    __shared__ uint32_t warp_tot[kCB / 32];
    __shared__ uint32_t list_n;

    const uint64_t n = *d_n;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t kNegInf = dev::ord_f32(-INFINITY);
    unsigned long long rows_local = 0;

    for (uint64_t base = uint64_t(blockIdx.x) * kCB; base < n; base += uint64_t(gridDim.x) * kCB) {
        const uint64_t idx = base + t;
        uint32_t pid = 0, len = 0;
        uint64_t off = 0;
        if (idx < n) {
            pid = cand_id(ids, keys, idx);
            // A passage that owns no token on a kept centroid (absent from every
            // kept centroid's posting list) has used == 0 and scores exactly 0
            // (pipeline.cpp:127-131): its codes need not be read at all.
            if (!owners || ((__ldg(owners + (pid >> 5)) >> (pid & 31)) & 1u)) {
                off = offsets[pid];
                len = doclens[pid];
            }
        }
        off_s[t] = off;
        // exclusive scan of len over the block
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += v;
        }
        if (lane == 31) warp_tot[warp] = incl;
        for (uint32_t j = 0; j < kAccPitch; ++j) acc_s[t * kAccPitch + j] = kNegInf;
        used_s[t] = 0;
        if (t == 0) list_n = 0;
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (uint32_t w = 0; w < kCB / 32; ++w) {
            if (w < warp) before += warp_tot[w];
            total += warp_tot[w];
        }
        start_s[t] = before + incl - len;
        if (t == 0) start_s[kCB] = total;
        __syncthreads();

        // sweep the flattened token range, 4 tokens per thread in flight
        for (uint32_t f0 = 0; f0 < total; f0 += 4 * kCB) {
            uint32_t code[4], cand[4];
            bool in[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t f = f0 + u * kCB + t;
                in[u] = f < total;
                uint32_t lo = 0, hi = kCB;
                while (hi - lo > 1) {
                    uint32_t mid = (lo + hi) >> 1;
                    if (start_s[mid] <= f) lo = mid; else hi = mid;
                }
                cand[u] = lo;
                code[u] = in[u] ? __ldg(codes + off_s[lo] + (f - start_s[lo])) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (in[u] && kept(keep_bits, code[u])) {
                    const uint32_t slot = atomicAdd(&list_n, 1u);
                    if (slot < kListCap) {
                        list_s[2 * slot] = cand[u];
                        list_s[2 * slot + 1] = code[u];
                    }
                }
            }
        }
        __syncthreads();
        const uint32_t nl = list_n;
        if (nl <= kListCap) {
            // fold the queued rows, 4 per warp in flight
            for (uint32_t e0 = warp; e0 < nl; e0 += 4 * (kCB / 32)) {
                float s[4];
                uint32_t cd[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * (kCB / 32);
                    cd[u] = e < nl ? list_s[2 * e] : 0u;
                    s[u] = e < nl ? __ldg(S + uint64_t(list_s[2 * e + 1]) * kScoresPitch + lane) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * (kCB / 32);
                    if (e < nl) {
                        if (lane < rows) atomicMax(&acc_s[cd[u] * kAccPitch + lane], dev::ord_f32(s[u]));
                        if (lane == 0) atomicAdd(&used_s[cd[u]], 1u);
                    }
                }
            }
            __syncthreads();
            if (idx < n) {
                const uint32_t u = used_s[t];
                float sc = 0.0f;
                if (u > 0)
                    for (uint32_t j = 0; j < rows; ++j)
                        sc = __fadd_rn(sc, dev::unord_f32(acc_s[t * kAccPitch + j]));
                out_keys[idx] = dev::make_key(sc, pid);
                if (out_scores) out_scores[idx] = sc;
                rows_local += u;
            }
        } else {
            // queue overflow (dense masks): score this block's passages warp-wide
            for (uint32_t c = warp; c < kCB && base + c < n; c += kCB / 32) {
                const uint32_t p = cand_id(ids, keys, base + c);
                uint32_t used;
                float sc = score_passage_warp<true>(codes, offsets[p], doclens[p], S, rows, keep_bits, &used);
                if (lane == 0) {
                    out_keys[base + c] = dev::make_key(sc, p);
                    if (out_scores) out_scores[base + c] = sc;
                    rows_local += used;
                }
            }
        }
        __syncthreads();
    }
    // block-level reduction of the gathered-row counter
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rows_local += __shfl_xor_sync(0xffffffffu, rows_local, o);
    dev::block_add_lane0(d_rows, rows_local);
}

// owners |= postings of every kept centroid: the passages that own at least
// one token on a kept centroid (IVF content invariant, index.cpp:64-83).  Each
// warp takes 32 keep-bit words (one per lane) and walks the set bits'
// posting lists cooperatively.
__global__ void kept_owners_kernel(const uint32_t* __restrict__ keep_bits, uint64_t K,
                                   const uint64_t* __restrict__ ivf_offsets,
                                   const uint32_t* __restrict__ postings, uint32_t* __restrict__ owners) {
    dev::pdl_wait();
    const uint32_t lane = dev::lane_id();
    const uint64_t words = (K + 31) / 32;
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t w0 = (uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < words;
         w0 += nw * 32) {
        const uint32_t mine = w0 + lane < words ? keep_bits[w0 + lane] : 0u;
        uint32_t nz = __ballot_sync(0xffffffffu, mine != 0);
        while (nz) {
            const int l = __ffs(nz) - 1;
            nz &= nz - 1;
            uint32_t bits = __shfl_sync(0xffffffffu, mine, l);
            while (bits) {
                const uint64_t c = (w0 + l) * 32 + (__ffs(bits) - 1);
                bits &= bits - 1;
                for (uint64_t j = ivf_offsets[c] + lane; j < ivf_offsets[c + 1]; j += 32) {
                    const uint32_t p = postings[j];
                    atomicOr(owners + (p >> 5), 1u << (p & 31));
                }
            }
        }
    }
}

// ---- stage 2 from the kept centroids' posting lists ------------------------------------
// Stage 2's score for candidate p is sum_i max over p's tokens on KEPT
// centroids of S[code][i] (0 if there is none, pipeline.cpp:127-131).  A max
// only needs the set of distinct kept codes of p, and p owns code c exactly
// when p is in postings(c) (IVF content invariant, index.cpp:64-83).  So the
// stage is driven by the kept centroids' posting lists, never reading codes:
//   keep_list        kept centroid ids + the total length of their lists;
//   ivf_accumulate   blocks over the kept lists: S[c] in registers (lane =
//                    query token), for each posting in C1 (slot_of[pid] =
//                    position in C1, written by the candidate compaction) one
//                    warp-wide atomicMax of the 32 order-preserving score
//                    images into acc[slot], the slot's used bit, and the
//                    posting's token multiplicity (index-derived ivf_mult)
//                    into the gathered-row counter;
//   stage2_finalize  thread per candidate: in-order fp32 sum of acc[slot]
//                    (exactly 0 when unused), the key, acc reset to 0, and
//                    the key histogram the stage-2 select starts from.
// Work is proportional to the kept (centroid, candidate) pairs.  When the kept
// lists are long (t_cs near -1 keeps most centroids) a warp-per-candidate
// pass over the codes (ci_all) takes over; the choice is made on the device.
__global__ void keep_list_kernel(const uint32_t* __restrict__ keep_bits, uint64_t K,
                                 const uint64_t* __restrict__ ivf_offsets, uint32_t* __restrict__ list,
                                 unsigned long long* __restrict__ counts /* [0] kept, [1] postings */) {
    dev::pdl_wait();
    fused::keep_list(blockIdx.x, gridDim.x, keep_bits, K, ivf_offsets, list, counts);
}

__device__ __forceinline__ bool use_lists(const unsigned long long* counts, uint64_t n1) {
    return counts[1] <= kListsPerCandidate * (n1 + 1024);
}

__global__ void __launch_bounds__(256)
ivf_accumulate_kernel(const uint32_t* __restrict__ list, const unsigned long long* __restrict__ counts,
                      const uint64_t* __restrict__ d_n1, const uint64_t* __restrict__ ivf_offsets,
                      const uint32_t* __restrict__ postings, const uint8_t* __restrict__ mult,
                      const uint32_t* __restrict__ cand_bits, const uint32_t* __restrict__ slot_of,
                      const float* __restrict__ S, uint32_t rows, const uint32_t* __restrict__ codes,
                      const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ doclens,
                      uint32_t* __restrict__ acc, uint32_t* __restrict__ used_bits,
                      unsigned long long* __restrict__ d_rows) {
    dev::pdl_wait();
    if (!use_lists(counts, *d_n1)) return;
    const uint64_t kept = counts[0];
    const uint32_t lane = dev::lane_id(), warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    unsigned long long rows_local = 0;
    // few kept centroids with long lists: every list is split over `parts` blocks
    const uint64_t parts = kept && gridDim.x > kept ? gridDim.x / kept : 1;
    for (uint64_t item = blockIdx.x; item < kept * parts; item += gridDim.x) {
        const uint64_t k = item % kept, part = item / kept;
        const uint32_t c = list[k];
        const uint32_t ord_s = dev::ord_f32(__ldg(S + uint64_t(c) * kScoresPitch + lane));
        const uint64_t e = ivf_offsets[c + 1];
        for (uint64_t j0 = ivf_offsets[c] + (part * nwarp + warp) * 32; j0 < e; j0 += parts * nwarp * 32) {
            const uint64_t j = j0 + lane;
            uint32_t slot = 0;
            bool in = false;
            if (j < e) {
                const uint32_t p = __ldg(postings + j);
                in = (__ldg(cand_bits + (p >> 5)) >> (p & 31)) & 1u;
                if (in) {
                    slot = __ldg(slot_of + p);
                    atomicOr(used_bits + (slot >> 5), 1u << (slot & 31));
                    uint32_t m = __ldg(mult + j);
                    if (m == 255) {  // saturated: recount from the codes
                        m = 0;
                        const uint64_t o = offsets[p];
                        for (uint32_t t = 0; t < doclens[p]; ++t) m += codes[o + t] == c;
                    }
                    rows_local += m;
                }
            }
            uint32_t b = __ballot_sync(0xffffffffu, in);
            while (b) {
                const int l = __ffs(b) - 1;
                b &= b - 1;
                const uint32_t s = __shfl_sync(0xffffffffu, slot, l);
                if (lane < rows) atomicMax(acc + uint64_t(s) * 32 + lane, ord_s);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rows_local += __shfl_xor_sync(0xffffffffu, rows_local, o);
    dev::block_add_lane0(d_rows, rows_local);
}

// Key histogram for the stage-2 select (select_top_hist): bucket = top 16
// key bits; warp-aggregated, the score-0 bucket of the all-masked candidates
// counted per block.
// Block sums (SelectHist::blk, one per 2048 buckets) are gathered per CTA in
// shared memory and flushed once at its end (hist_flush).
__device__ __forceinline__ void hist_key(SelectHist* hs, uint64_t key, bool valid, uint32_t* zeros,
                                         uint32_t* blk_s) {
    const uint32_t lane = dev::lane_id();
    const uint32_t b = valid ? uint32_t(key >> kHistShift) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    if (valid && lane == uint32_t(__ffs(peers) - 1)) {
        if (b == kHistZeroBucket) atomicAdd(zeros, uint32_t(__popc(peers)));
        else {
            atomicAdd(&hs->hist[dev::hist_slot(b)], uint32_t(__popc(peers)));
            atomicAdd(&blk_s[b >> 11], uint32_t(__popc(peers)));
        }
    }
}

__device__ __forceinline__ void hist_flush(SelectHist* hs, uint32_t zeros, const uint32_t* blk_s) {
    if (threadIdx.x == 0 && zeros) {
        atomicAdd(&hs->hist[dev::hist_slot(kHistZeroBucket)], zeros);
        atomicAdd(&hs->blk[kHistZeroBucket >> 11], zeros);
    }
    if (threadIdx.x < 32 && blk_s[threadIdx.x]) atomicAdd(&hs->blk[threadIdx.x], blk_s[threadIdx.x]);
}

__device__ __forceinline__ void stage2_finalize(const uint32_t* __restrict__ c1, uint64_t n, uint32_t rows,
                                                uint32_t* __restrict__ acc, const uint32_t* __restrict__ used_bits,
                                                uint64_t* __restrict__ keys_out, SelectHist* __restrict__ hs) {
    __shared__ uint32_t zeros, blk_s[32];
    if (threadIdx.x == 0) zeros = 0;
    if (threadIdx.x < 32) blk_s[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t i0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~31ull; i0 < n;
         i0 += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = i0 + dev::lane_id();
        float sc = 0.0f;
        uint64_t key = 0;
        if (i < n && ((used_bits[i >> 5] >> (i & 31)) & 1u)) {
            uint4* a4 = reinterpret_cast<uint4*>(acc + i * 32);
            uint32_t v[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 x = a4[q];
                v[4 * q] = x.x, v[4 * q + 1] = x.y, v[4 * q + 2] = x.z, v[4 * q + 3] = x.w;
                a4[q] = make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int q = 0; q < 32; ++q)
                if (uint32_t(q) < rows) sc = __fadd_rn(sc, dev::unord_f32(v[q]));
        }
        if (i < n) {
            key = dev::make_key(sc, c1[i]);
            keys_out[i] = key;
        }
        hist_key(hs, key, i < n, &zeros, blk_s);
    }
    __syncthreads();
    hist_flush(hs, zeros, blk_s);
}

// fallback when the kept lists are long: warp per candidate over its codes
__device__ __forceinline__ void ci_all(const uint32_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                                       const uint32_t* __restrict__ doclens, const float* __restrict__ S,
                                       uint32_t rows, const uint32_t* __restrict__ c1, uint64_t n,
                                       const uint32_t* __restrict__ keep_bits, uint64_t* __restrict__ keys_out,
                                       unsigned long long* __restrict__ d_rows, SelectHist* __restrict__ hs) {
    const uint32_t lane = dev::lane_id();
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    unsigned long long rows_local = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const uint32_t pid = c1[i];
        uint32_t used;
        const float total = score_passage_warp<true>(codes, offsets[pid], doclens[pid], S, rows, keep_bits, &used);
        if (lane == 0) {
            const uint64_t key = dev::make_key(total, pid);
            keys_out[i] = key;
            atomicAdd(&hs->hist[dev::hist_slot(uint32_t(key >> kHistShift))], 1u);
            atomicAdd(&hs->blk[uint32_t(key >> kHistShift) >> 11], 1u);
        }
        rows_local += used;
    }
    dev::block_add_lane0(d_rows, rows_local);
}

// The stage-2 keys: the list finalize or, when the kept lists are long, the
// per-candidate fallback — one launch, the branch taken on the device.
__global__ void __launch_bounds__(256)
stage2_keys_kernel(const uint32_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                   const uint32_t* __restrict__ doclens, const float* __restrict__ S, uint32_t rows,
                   const uint32_t* __restrict__ c1, const uint64_t* __restrict__ d_n1,
                   const unsigned long long* __restrict__ counts, const uint32_t* __restrict__ keep_bits,
                   uint32_t* __restrict__ acc, const uint32_t* __restrict__ used_bits,
                   uint64_t* __restrict__ keys_out, unsigned long long* __restrict__ d_rows,
                   SelectHist* __restrict__ hs) {
    dev::pdl_wait();
    const uint64_t n = *d_n1;
    if (use_lists(counts, n))
        stage2_finalize(c1, n, rows, acc, used_bits, keys_out, hs);
    else
        ci_all(codes, offsets, doclens, S, rows, c1, n, keep_bits, keys_out, d_rows, hs);
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

void kept_owners(const IndexView& ix, const uint32_t* d_keep_bits, uint32_t* d_owners, cudaStream_t st) {
    const uint64_t tasks = ((ix.K + 31) / 32 + 31) / 32;  // one warp per 32 keep words
    uint64_t blocks = (tasks + 7) / 8;
    if (blocks == 0) blocks = 1;
    ::plaid::launch::pdl(kept_owners_kernel, uint32_t(blocks), 256, 0, st, d_keep_bits, ix.K, ix.ivf_offsets, ix.ivf_postings,
                                                         d_owners);
    count_launch();
}

void stage2_masked(const IndexView& ix, const float* d_scores, uint32_t rows, const uint32_t* d_c1,
                   const uint64_t* d_n1, uint64_t nmax, const uint32_t* d_keep_bits, const uint32_t* d_cand_bits,
                   uint32_t* d_used_bits, uint32_t* d_kept_list, const uint32_t* d_slot_of, uint32_t* d_acc,
                   unsigned long long* d_counts2, uint64_t* d_out_keys, unsigned long long* d_rows,
                   SelectHist* d_hist, bool kept_ready, cudaStream_t st) {
    const uint32_t sms = uint32_t(sm_count());
    if (!kept_ready) {
        ::plaid::launch::pdl(keep_list_kernel, keep_list_blocks(ix.K), 256, 0, st, d_keep_bits, ix.K, ix.ivf_offsets,
                             d_kept_list, d_counts2);
        count_launch();
    }
    if (nmax == 0) return;
    uint64_t sb = (nmax + 255) / 256;
    if (sb > uint64_t(sms) * 8) sb = uint64_t(sms) * 8;
    ::plaid::launch::pdl(ivf_accumulate_kernel, sms * 8, 256, 0, st, d_kept_list, d_counts2, d_n1, ix.ivf_offsets,
                         ix.ivf_postings, ix.ivf_mult, d_cand_bits, d_slot_of, d_scores, rows, ix.codes, ix.offsets,
                         ix.doclens, d_acc, d_used_bits, d_rows);
    count_launch();
    if (sb < uint64_t(sms) * 2) sb = uint64_t(sms) * 2;  // the fallback's warp-per-candidate width
    ::plaid::launch::pdl(stage2_keys_kernel, uint32_t(sb), 256, 0, st, ix.codes, ix.offsets, ix.doclens, d_scores, rows,
                         d_c1, d_n1, d_counts2, d_keep_bits, d_acc, d_used_bits, d_out_keys, d_rows, d_hist);
    count_launch();
}

void centroid_interaction(const IndexView& ix, const float* d_scores, uint32_t rows,
                          const uint32_t* d_ids, const uint64_t* d_keys, const uint64_t* d_n,
                          uint64_t nmax, const uint32_t* d_keep_bits, const uint32_t* d_owners,
                          uint64_t* d_out_keys, float* d_out_scores, unsigned long long* d_rows,
                          cudaStream_t st, uint32_t* d_out_len, uint64_t* d_out_off) {
    if (nmax == 0) return;
    if (d_keep_bits && d_out_len) fail_cuda_driver(1, "centroid_interaction: (len, off) outputs are unmasked-only");
    if (d_keep_bits) {
        uint64_t blocks = (nmax + kCB - 1) / kCB;
        const uint64_t cap = uint64_t(sm_count()) * 4;
        if (blocks > cap) blocks = cap;
        ::plaid::launch::pdl(ci_masked_flat_kernel, uint32_t(blocks), kCB, 0, st, 
            ix.codes, ix.offsets, ix.doclens, d_scores, rows, d_ids, d_keys, d_n, d_keep_bits, d_owners,
            d_out_keys, d_out_scores, d_rows);
    } else {
        uint64_t blocks = (nmax + 7) / 8;
        const uint64_t cap = uint64_t(sm_count()) * 8;
        if (blocks > cap) blocks = cap;
        ::plaid::launch::pdl(ci_warp_kernel, uint32_t(blocks), 256, 0, st, ix.codes, ix.offsets, ix.doclens, d_scores,
                                                        rows, d_ids, d_keys, d_n, d_keep_bits,
                                                        d_out_keys, d_out_scores, d_rows, d_out_len, d_out_off);
    }
    count_launch();
}

}  // namespace launch
}  // namespace plaid
