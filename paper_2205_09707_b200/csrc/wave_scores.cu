// wave_scores.cu — throughput-mode stage 1: S_cq = Q . C^T for a wave of
// queries on the 5th-gen tensor cores, four queries per pass over C.
// Replaces compute_centroid_scores (pipeline.cpp:26-50) for batched search
// and fuses its two consumers: the per-token top-nprobe lists
// (pipeline.cpp:52-88) and the t_cs keep bits (pipeline.cpp:90-110).
//
// Orientation: M = 128 query tokens (4 queries x 32 rows, TMEM lane quarter q
// = query q of the group), N = 128 centroids per tile, K = 128 dims.
//   A = [Q_hi | Q_lo] of the group in TMEM (256 columns, loaded once per
//       group), B = the centroid tile from shared memory: the raw fp32 TMA box
//       IS C_hi (the tensor core truncates fp32 operands to tf32), and
//       converter warps write C_lo = C - C_hi beside it in the same swizzled
//       layout (truncated to tf32 by the tensor core in turn).
//   D = Q_hi.C_hi + Q_lo.C_hi + Q_hi.C_lo (3xTF32, fp32 accumulate, ~2e-6
//       absolute on unit-vector dots), two 128-column accumulators.
// A TMA box is 128 centroids x 32 dims (16 KB, SWIZZLE_128B: K-major rows of
// 128 B), i.e. exactly one K-chunk of the B operand; a tile is 4 boxes.
//
// Roles (persistent, one CTA per SM, 16 warps):
//   warp 0      TMA producer, 8-box ring (2 tiles, 128 KB in flight);
//   warp 1      MMA issuer: per chunk 12 MMAs (M=128, N=128, K=8) issued by
//               the converged warp in one asm block, commits release the
//               ring slots; one commit per tile to the accumulator;
//   warps 4-7   converters (thread = centroid row of a box) and, at every
//               group boundary, the A loaders (thread = query token row);
//   warps 8-15  epilogue, two groups taking alternate tiles: tcgen05.ld,
//               lane = query token, so every S row store (centroid c, the 32
//               tokens) is one coalesced 128-B line; keep bit = any lane's
//               score >= t_cs (one vote per centroid); per-lane top-NP
//               (score, id) list of the token, flushed per group into the
//               query's partial lists [grid x 2][32][NP] (key 0 = empty).
// Work order: groups outer, this CTA's tiles inner, every other group walking
// the tiles backwards so the tiles read last are read first again (some
// L2 hits on the 134 MB table).
// Traffic per query at K = 2^18: C / 4 = 32 MB read + 32 MB of S written
// (the S rows are read back by stages 2-3), so the pass is HBM-bound at
// ~64 MB per query; tensor work 6.4 GFLOP per query.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"
#include "tc.cuh"

namespace plaid {
namespace {

constexpr int kThreads = 512;
constexpr uint32_t kBoxBytes = 128 * 128;  // 128 centroids x 32 fp32
constexpr int kRaw = 8;                    // TMA ring (boxes)
constexpr int kLo = 4;                     // C_lo ring: one tile
constexpr uint32_t kOffRaw = 0;
constexpr uint32_t kOffLo = kOffRaw + kRaw * kBoxBytes;
constexpr uint32_t kOffBar = kOffLo + kLo * kBoxBytes;
constexpr uint32_t kNumBars = 2 * kRaw + 2 * kLo + 4 + 2;
constexpr uint32_t kOffMisc = kOffBar + kNumBars * 8;
constexpr uint32_t kOffStage = (kOffMisc + 16 + 15) / 16 * 16;  // epilogue: 8 warps x 32 lanes x 33 f32
constexpr uint32_t kSmemBytes = kOffStage + 8 * 32 * 33 * 4 + 1024;
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
constexpr uint32_t kTmemCols = 512;  // [0,256) two accumulators, [256,384) Q_hi, [384,512) Q_lo
constexpr uint32_t kColA = 256;
constexpr uint32_t kIdesc = tc::idesc_tf32(128, 128);

// chunk of 32 dims: 4 k-steps x (Q_hi.C_hi, Q_lo.C_hi, Q_hi.C_lo) into d.
// One asm block from the converged warp (elect.sync inside).
__device__ __forceinline__ void mma_chunk(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t braw, uint64_t blo,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred e, pa, pt;\n\t"
        ".reg .b32 rx, h1, h2, h3, l1, l2, l3;\n\t"
        ".reg .b64 r1, r2, r3, o1, o2, o3;\n\t"
        "elect.sync rx|e, 0xffffffff;\n\t"
        "setp.ne.b32 pa, %5, 0;\n\t"
        "setp.eq.b32 pt, %5, %5;\n\t"
        "add.u32 h1, %1, 8;\n\t"
        "add.u32 h2, %1, 16;\n\t"
        "add.u32 h3, %1, 24;\n\t"
        "add.u32 l1, %2, 8;\n\t"
        "add.u32 l2, %2, 16;\n\t"
        "add.u32 l3, %2, 24;\n\t"
        "add.s64 r1, %3, 2;\n\t"
        "add.s64 r2, %3, 4;\n\t"
        "add.s64 r3, %3, 6;\n\t"
        "add.s64 o1, %4, 2;\n\t"
        "add.s64 o2, %4, 4;\n\t"
        "add.s64 o3, %4, 6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %6, pa;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h1], r1, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [l1], r1, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h1], o1, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h2], r2, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [l2], r2, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h2], o2, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h3], r3, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [l3], r3, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h3], o3, %6, pt;\n\t"
        "}" ::"r"(d),
        "r"(ahi), "r"(alo), "l"(braw), "l"(blo), "r"(accumulate), "r"(kIdesc)
        : "memory");
}

// C_lo = C - C_hi exactly (fp32), left for the tensor core to truncate: the
// dropped bits are < 2^-22 |c| per element (a bias below 3e-7 on a unit dot
// product, far inside the 3xTF32 error), and the converter saves the
// rounding's two ALU operations per element — the ALU pipe, not the tensor
// core or HBM, limited this kernel.
__device__ __forceinline__ uint32_t lo_trunc(uint32_t x) {
    return __float_as_uint(__fsub_rn(__uint_as_float(x), __uint_as_float(tc::split_hi(x))));
}

// 0xFFFFFFFF when a >= b (a > b), else 0: one FSET instead of a compare and a select
__device__ __forceinline__ uint32_t fset_ge(float a, float b) {
    uint32_t r;
    asm("set.ge.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint32_t fset_gt(float a, float b) {
    uint32_t r;
    asm("set.gt.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
    return r;
}

template <int NP>
__global__ void __launch_bounds__(kThreads, 1)
wave_scores_kernel(const __grid_constant__ CUtensorMap cmap, uint64_t K, const float* __restrict__ Q, uint32_t nq,
                   uint32_t rows, float t_cs, float* __restrict__ S, uint64_t s_stride, uint32_t* __restrict__ keep,
                   uint64_t keep_stride, uint64_t* __restrict__ partial, uint64_t partial_stride) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t base = tc::smem_u32(smem);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = base + kOffBar;
    auto raw_full = [&](uint32_t s) { return bar0 + 8u * s; };
    auto raw_empty = [&](uint32_t s) { return bar0 + 8u * (kRaw + s); };
    auto lo_full = [&](uint32_t s) { return bar0 + 8u * (2 * kRaw + s); };
    auto lo_empty = [&](uint32_t s) { return bar0 + 8u * (2 * kRaw + kLo + s); };
    auto tfull = [&](uint32_t a) { return bar0 + 8u * (2 * kRaw + 2 * kLo + a); };
    auto tempty = [&](uint32_t a) { return bar0 + 8u * (2 * kRaw + 2 * kLo + 2 + a); };
    const uint32_t a_full = bar0 + 8u * (2 * kRaw + 2 * kLo + 4);
    const uint32_t a_empty = a_full + 8u;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffMisc);

    const uint64_t ntiles = (K + 127) / 128;
    const uint32_t my_tiles = uint32_t((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);  // grid <= ntiles
    const uint32_t groups = (nq + 3) / 4;
    const uint32_t nitems = groups * my_tiles;
    // item -> tile: every other group walks this CTA's tiles backwards
    auto tile_of = [&](uint32_t it) -> uint64_t {
        const uint32_t g = it / my_tiles, i = it % my_tiles;
        const uint32_t j = (g & 1) ? my_tiles - 1 - i : i;
        return blockIdx.x + uint64_t(j) * gridDim.x;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kRaw; ++s) {
            tc::mbar_init(raw_full(s), 1);
            tc::mbar_init(raw_empty(s), 4 + 1);  // 4 converter warps + the MMA commit
        }
        for (int s = 0; s < kLo; ++s) {
            tc::mbar_init(lo_full(s), 4);
            tc::mbar_init(lo_empty(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(tfull(a), 1);
            tc::mbar_init(tempty(a), 4);
        }
        tc::mbar_init(a_full, 4);
        tc::mbar_init(a_empty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&cmap)) : "memory");
    }
    // C is index data: the producer starts streaming it before waiting on the
    // previous kernel (the wave prologue); everyone else waits first
    auto issue_box = [&](uint32_t gb) {
        const uint32_t s = gb % kRaw;
        tc::mbar_wait(raw_empty(s), ((gb / kRaw) & 1) ^ 1);
        tc::mbar_expect_tx(raw_full(s), kBoxBytes);
        const uint64_t t = tile_of(gb / 4);
        tc::tma_load_2d(base + kOffRaw + s * kBoxBytes, &cmap, int((gb % 4) * 32), int(t * 128), raw_full(s));
    };
    const uint32_t nboxes = nitems * 4;
    const uint32_t pre = nboxes < uint32_t(kRaw) ? nboxes : uint32_t(kRaw);
    __syncthreads();  // barrier init visible
    if (threadIdx.x == 0)
        for (uint32_t g = 0; g < pre; ++g) issue_box(g);
    if (warp != 0) dev::pdl_wait();
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0)
            for (uint32_t gb = pre; gb < nboxes; ++gb) issue_box(gb);
    } else if (warp == 1) {
        // ---------------- MMA issuer
        for (uint32_t it = 0; it < nitems; ++it) {
            const uint32_t g = it / my_tiles, i = it % my_tiles;
            if (i == 0) {
                tc::mbar_wait(a_full, g & 1);
                tc::fence_after();
            }
            const uint32_t acc = it & 1, u = it >> 1;
            tc::mbar_wait(tempty(acc), (u & 1) ^ 1);
            tc::fence_after();
            const uint32_t d = tmem + acc * 128;
            for (uint32_t kc = 0; kc < 4; ++kc) {
                const uint32_t gb = it * 4 + kc, s = gb % kRaw;
                tc::mbar_wait(raw_full(s), (gb / kRaw) & 1);
                tc::mbar_wait(lo_full(kc), it & 1);
                tc::fence_after();
                mma_chunk(d, tmem + kColA + kc * 32, tmem + kColA + 128 + kc * 32,
                          tc::desc_sw128(base + kOffRaw + s * kBoxBytes), tc::desc_sw128(base + kOffLo + kc * kBoxBytes),
                          kc);
                tc::commit_warp(raw_empty(s));
                tc::commit_warp(lo_empty(kc));
                __syncwarp();
            }
            tc::commit_warp(tfull(acc));
            if (i == my_tiles - 1) tc::commit_warp(a_empty);
            __syncwarp();
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- converters / A loaders: lane quarter q = warp - 4
        const uint32_t q = warp - 4, r = q * 32 + lane;
        for (uint32_t it = 0; it < nitems; ++it) {
            const uint32_t g = it / my_tiles, i = it % my_tiles;
            for (uint32_t kc = 0; kc < 4; ++kc) {
                const uint32_t gb = it * 4 + kc, s = gb % kRaw;
                tc::mbar_wait(raw_full(s), (gb / kRaw) & 1);
                tc::mbar_wait(lo_empty(kc), (it & 1) ^ 1);
                // row r's 8 granules (swizzled: granule j at j ^ (r & 7)), lo to the same spots
                const uint4* src = reinterpret_cast<const uint4*>(smem + kOffRaw + s * kBoxBytes + r * 128);
                uint4* dst = reinterpret_cast<uint4*>(smem + kOffLo + kc * kBoxBytes + r * 128);
                // granule order rotated by row (j ^ (r & 7)): conflict-free LDS/STS.128
                uint4 v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = src[j ^ (lane & 7)];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    dst[j ^ (lane & 7)] = make_uint4(lo_trunc(v[j].x), lo_trunc(v[j].y), lo_trunc(v[j].z),
                                                     lo_trunc(v[j].w));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(lo_full(kc));
                    tc::mbar_arrive(raw_empty(s));
                }
            }
            if (i == 0) {
                // A of group g (after converting its first tile, so the MMA's
                // wait for A is the only bubble at a group boundary)
                // Q rows of the group, two 32-dim chunks per round trip; the
                // first two are in flight before A is free (the MMA waits for
                // A at every group boundary: the reload is the bubble).  A_hi
                // is the raw fp32 row (the tensor core truncates it to tf32)
                const uint32_t qi = g * 4 + q;
                const bool live = qi < nq && lane < rows;
                const uint4* qr = reinterpret_cast<const uint4*>(Q + (uint64_t(qi) * rows + lane) * 128);
                auto load2 = [&](uint32_t kc, uint32_t (&x)[64]) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint4 v = live ? __ldg(qr + kc * 8 + j) : make_uint4(0, 0, 0, 0);
                        x[4 * j] = v.x, x[4 * j + 1] = v.y, x[4 * j + 2] = v.z, x[4 * j + 3] = v.w;
                    }
                };
                auto store2 = [&](uint32_t kc, uint32_t (&x)[64]) {
                    const uint32_t col = tmem + ((q * 32) << 16) + kColA + kc * 32;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t (&v)[32] = *reinterpret_cast<uint32_t(*)[32]>(&x[32 * h]);
                        tc::tmem_st32(col + 32 * h, v);
                        tc::tmem_st_wait();  // v is overwritten next
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = tc::split_lo(v[e]);
                        tc::tmem_st32(col + 128 + 32 * h, v);
                        tc::tmem_st_wait();
                    }
                };
                uint32_t xq[64];
                load2(0, xq);
                if (g > 0) tc::mbar_wait(a_empty, (g - 1) & 1);
                tc::fence_after();
                store2(0, xq);
                load2(2, xq);
                store2(2, xq);
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(a_full);
            }
        }
    } else if (warp >= 8) {
        // ---------------- epilogue: group grp takes the items of parity grp
        const uint32_t ew = warp - 8, grp = ew >> 2, q = warp & 3;
        const bool tok = lane < rows;
        uint32_t* stage = reinterpret_cast<uint32_t*>(smem + kOffStage) + (ew * 32 + lane) * 33;
        float top_s[NP];
        uint32_t top_i[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) top_s[j] = -INFINITY, top_i[j] = 0;
        for (uint32_t it = 0; it < nitems; ++it) {
            const uint32_t g = it / my_tiles, i = it % my_tiles;
            const uint32_t qi = g * 4 + q;
            const bool live = qi < nq;
            if ((it & 1) == grp) {
                const uint32_t acc = grp, u = it >> 1;
                tc::mbar_wait(tfull(acc), u & 1);
                tc::fence_after();
                const uint64_t t = tile_of(it);
                float* Sq = S + uint64_t(qi) * s_stride;
#pragma unroll 1
                for (uint32_t jb = 0; jb < 4; ++jb) {
                    uint32_t raw[32];
                    tc::tmem_ld32(tmem + ((q * 32) << 16) + acc * 128 + jb * 32, raw);
                    tc::tmem_ld_wait();
                    if (jb == 3) {
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(tempty(acc));
                    }
                    const uint64_t c0 = t * 128 + jb * 32;
                    if (!live || c0 >= K) continue;
                    const uint32_t nv = K - c0 < 32 ? uint32_t(K - c0) : 32u;
                    // per lane (= token) bit masks over the 32 centroids, then one
                    // OR-reduction across the tokens for the keep word: the ALU
                    // pipe, not HBM, was the limit with a vote per centroid
                    const float thr0 = top_s[NP - 1];
                    uint32_t km = 0, cm = 0;
                    float* Srow = Sq + c0 * kScoresPitch + lane;
                    if (nv == 32) {  // whole tile column block: no per-centroid bound checks
#pragma unroll
                        for (int r = 0; r < 32; ++r) {
                            const float v = __uint_as_float(raw[r]);
                            __stcs(Srow + r * kScoresPitch, v);  // evict-first: keep L2 for C's reuse
                            km |= fset_ge(v, t_cs) & (1u << r);
                            cm |= fset_gt(v, thr0) & (1u << r);
                        }
                    } else {
#pragma unroll
                        for (int r = 0; r < 32; ++r) {
                            const float v = __uint_as_float(raw[r]);
                            if (uint32_t(r) < nv) __stcs(Srow + r * kScoresPitch, v);
                            km |= fset_ge(v, t_cs) & (1u << r);
                            cm |= fset_gt(v, thr0) & (1u << r);
                        }
                    }
                    const uint32_t vmask = nv == 32 ? 0xFFFFFFFFu : (1u << nv) - 1u;
                    const uint32_t kw = __reduce_or_sync(0xffffffffu, tok ? km : 0u);
                    uint32_t cand = tok ? cm & vmask : 0u;
                    if (lane == 0) keep[uint64_t(qi) * keep_stride + (c0 >> 5)] = kw & vmask;
                    // inserts (centroids arrive in increasing id order within a
                    // tile; strict > keeps the lower id on ties).  Many
                    // candidates (a group's first tiles, lists still short):
                    // one static pass over the 32 values; few: extract each
                    auto insert = [&](float sc, uint32_t id) {
#pragma unroll
                        for (int j = NP - 1; j > 0; --j) {
                            const bool up = sc > top_s[j - 1], here = sc > top_s[j];
                            top_i[j] = up ? top_i[j - 1] : (here ? id : top_i[j]);
                            top_s[j] = up ? top_s[j - 1] : (here ? sc : top_s[j]);
                        }
                        if (sc > top_s[0]) top_s[0] = sc, top_i[0] = id;
                    };
                    if (__any_sync(0xffffffffu, __popc(cand) > 4)) {
#pragma unroll
                        for (int r = 0; r < 32; ++r) {
                            const float sc = __uint_as_float(raw[r]);
                            if (((cand >> r) & 1u) && sc > top_s[NP - 1]) insert(sc, uint32_t(c0 + r));
                        }
                        cand = 0;
                    }
                    if (__any_sync(0xffffffffu, cand != 0u)) {  // stage the row for the extractions
#pragma unroll
                        for (int r = 0; r < 32; ++r) stage[r] = raw[r];
                        __syncwarp();
                    }
                    while (cand) {
                        const int r = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const float sc = __uint_as_float(stage[r]);
                        if (sc > top_s[NP - 1]) {
                            const uint32_t id = uint32_t(c0 + r);
#pragma unroll
                            for (int j = NP - 1; j > 0; --j) {
                                const bool up = sc > top_s[j - 1], here = sc > top_s[j];
                                top_i[j] = up ? top_i[j - 1] : (here ? id : top_i[j]);
                                top_s[j] = up ? top_s[j - 1] : (here ? sc : top_s[j]);
                            }
                            if (sc > top_s[0]) top_s[0] = sc, top_i[0] = id;
                        }
                    }
                }
            }
            if (i == my_tiles - 1) {
                // end of group g: this group's list for (query, token)
                if (live) {
                    uint64_t* po = partial + uint64_t(qi) * partial_stride + ((blockIdx.x * 2 + grp) * 32 + lane) * NP;
#pragma unroll
                    for (int j = 0; j < NP; ++j)
                        po[j] = (tok && top_s[j] != -INFINITY) ? dev::make_key(top_s[j], top_i[j]) : 0ull;
                }
#pragma unroll
                for (int j = 0; j < NP; ++j) top_s[j] = -INFINITY, top_i[j] = 0;
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
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
void launch_wave(const CUtensorMap& map, uint64_t K, const float* d_q, uint32_t nq, uint32_t rows, float t_cs,
                 float* d_S, uint64_t s_stride, uint32_t* d_keep, uint64_t keep_stride, uint64_t* d_partial,
                 uint64_t partial_stride, uint32_t grid, cudaStream_t st) {
    static launch::PerDeviceOnce configured;
    if (configured.first())
        cudaFuncSetAttribute(wave_scores_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    ::plaid::launch::pdl(wave_scores_kernel<NP>, grid, kThreads, kSmemBytes, st, map, K, d_q, nq, rows, t_cs, d_S,
                         s_stride, d_keep, keep_stride, d_partial, partial_stride);
    launch::count_launch();
}

}  // namespace

namespace launch {

void make_wave_tensor_map(const IndexView& ix, void* out_map) {
    CUtensorMap* map = static_cast<CUtensorMap*>(out_map);
    // 2-D view (128 fp32 dims, K centroids): box = 32 dims x 128 centroids,
    // 128-B rows, SWIZZLE_128B (K-major B operand of one 32-dim chunk)
    const cuuint64_t dims[2] = {128, cuuint64_t(ix.K)};
    const cuuint64_t strides[1] = {128 * sizeof(float)};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t estr[2] = {1, 1};
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<EncodeFn>(fn);
    }();
    if (!encode) fail_cuda_driver(int(CUDA_ERROR_NOT_FOUND), "cuGetProcAddress(cuTensorMapEncodeTiled)");
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ix.centroids), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail_cuda_driver(int(r), "cuTensorMapEncodeTiled");
}

uint32_t wave_scores_lists(const IndexView& ix) {
    const uint64_t ntiles = (ix.K + 127) / 128;
    const uint64_t g = ntiles < uint64_t(sm_count()) ? ntiles : uint64_t(sm_count());
    return uint32_t(g ? g : 1) * 2;
}

uint32_t wave_scores(const void* cmap, const IndexView& ix, const float* d_q, uint32_t nq, uint32_t rows, float t_cs,
                     uint32_t np_bucket, float* d_S, uint64_t s_stride, uint32_t* d_keep, uint64_t keep_stride,
                     uint64_t* d_partial, uint64_t partial_stride, cudaStream_t st) {
    const CUtensorMap& map = *static_cast<const CUtensorMap*>(cmap);
    const uint32_t lists = wave_scores_lists(ix), grid = lists / 2;
    switch (np_bucket) {
        case 1: launch_wave<1>(map, ix.K, d_q, nq, rows, t_cs, d_S, s_stride, d_keep, keep_stride, d_partial, partial_stride, grid, st); break;
        case 2: launch_wave<2>(map, ix.K, d_q, nq, rows, t_cs, d_S, s_stride, d_keep, keep_stride, d_partial, partial_stride, grid, st); break;
        case 4: launch_wave<4>(map, ix.K, d_q, nq, rows, t_cs, d_S, s_stride, d_keep, keep_stride, d_partial, partial_stride, grid, st); break;
        case 8: launch_wave<8>(map, ix.K, d_q, nq, rows, t_cs, d_S, s_stride, d_keep, keep_stride, d_partial, partial_stride, grid, st); break;
        default: fail_cuda_driver(1, "wave S_cq supports nprobe <= 8");
    }
    return lists;
}

}  // namespace launch
}  // namespace plaid
