// rank128.cu — stage 4 for d = 128 (pipeline.cpp:165-225): residual
// decompression (residual_codec.cpp:97-132) fused with exact MaxSim
// (maxsim.cpp:66-104) over the finalists' tokens as ONE packed stream.
//
// The finalists' tokens are laid end to end (finalist p's tokens start at
// pref[p], an exclusive scan of their doclens) and processed in full 64-token
// tiles, so no lane idles on a passage tail and the grid is sized by tokens:
//   K1 finalist_scan   one CTA: pref[] over the (<= 16384) finalists and the
//                      index-token base of each;
//   K2 stream_fused    persistent CTAs, warp-specialised around a 2-deep ring
//                      of tiles in shared memory:
//                      * 2 producer warps decompress the next tile: centroid
//                        rows by cp.async (lane = 16 bytes of a row), the
//                        token's packed residual row in registers, then lane =
//                        token: v = C + w[idx], the in-order fp64 norm and
//                        v *= inv — bit for bit the reference's arithmetic;
//                      * 4 consumer warps score the ready tile: lane = token
//                        (two per lane), warp w = query tokens 8w..8w+7,
//                        in-order fp32 dot chains with FMUL2 products over
//                        query pairs and separately rounded adds; then a
//                        segmented max across the lanes of each finalist and
//                        one atomicMax per (finalist, query) into run[p][i]
//                        (order-preserving uint image of the float);
//   K3 finalize        thread per finalist: score = in-order fp32 sum of
//                      run[p][i], the 64-bit (score, pid) key, run reset to 0.
// HBM traffic per finalist token: 4 B code + 16*b B residuals + the 512-byte
// centroid row (rows shared by tokens hit L2); the decompressed rows never
// leave shared memory.  The bound is the exact fp32 issue rate (FMA and
// tensor cores would change the rounding), see DESIGN.md §3.
#include <cuda_bf16.h>
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

constexpr uint32_t kPitch = 132;   // floats per shared-memory row (conflict-free LDS.128 both ways)
constexpr uint32_t kTile = 64;     // stream tokens per tile (two per consumer lane)
constexpr uint32_t kConsumers = 4; // x 8 query tokens = 32
constexpr uint32_t kProducers = 2; // x 32 tokens = one tile
constexpr uint32_t kFusedThreads = (kConsumers + kProducers) * 32;
constexpr uint32_t kSmemFloats = 16 * 128 * 2 + 2 * kTile * kPitch;  // query pairs + 2 tiles

// Debug timeline (PLAID_RANK_DBG=1): globaltimer stamps of CTA 0's tiles
// [event][tile]: 0 producer start, 1 producer rows landed, 2 producer done,
// 3 consumer start, 4 consumer done (read with plaid_debug_rank_trace).
__device__ unsigned long long g_rank_trace[5 * 64];
__device__ __forceinline__ void rank_stamp(uint32_t dbg, int ev, uint32_t k) {
    if (dbg && blockIdx.x == 0 && k < 64 && dev::lane_id() == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_rank_trace[ev * 64 + k] = t;
    }
}

struct Weights16 {
    float w[16];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint32_t finalist_pid(const uint32_t* ids, const uint64_t* keys, uint64_t p) {
    return ids ? ids[p] : dev::key_id(keys[p]);
}

// ---- K1: exclusive scan of finalist lengths -----------------------------------------
__global__ void __launch_bounds__(1024)
finalist_scan_kernel(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ keys,
                     const uint64_t* __restrict__ d_n, const uint32_t* __restrict__ doclens,
                     const uint64_t* __restrict__ offsets, uint32_t* __restrict__ pref,
                     uint64_t* __restrict__ fin_base, uint64_t* __restrict__ tokens, uint32_t* __restrict__ run_p0) {
    dev::pdl_wait();
    fused::finalist_scan(ids, keys, uint32_t(*d_n), doclens, offsets, pref, fin_base, tokens, run_p0);
}

// Warp-cooperative: the finalist of stream token g (this lane's) for a
// 32-token run starting at g0.  A 32-ary search finds p0 (pref[p0] <= g0 <
// pref[p0 + 1]) in ceil(log32 n) rounds of one load per lane; the run's tokens
// then lie in finalists p0 .. p0 + 31 (each has >= 1 token), whose ends one
// load per lane brings in.
__device__ __forceinline__ uint32_t run_finalists(const uint32_t* __restrict__ pref, uint32_t n, uint32_t g0,
                                                  uint32_t g) {
    const uint32_t lane = dev::lane_id();
    uint32_t lo = 0, span = n;  // pref[lo] <= g0 < pref[lo + span]
    while (span > 1) {
        const uint32_t step = (span + 31) / 32;
        const uint32_t probe = lo + lane * step;
        const bool le = probe < lo + span && __ldg(pref + probe) <= g0;
        const uint32_t last = 31 - __clz(__ballot_sync(0xffffffffu, le));  // lane 0 always qualifies
        lo += last * step;
        span = (last + 1) * step <= span ? step : span - last * step;
    }
    const uint32_t e = lo + 1 + lane <= n ? __ldg(pref + lo + 1 + lane) : 0xFFFFFFFFu;  // end of finalist lo + lane
    uint32_t p = lo;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) p += __shfl_sync(0xffffffffu, e, j) <= g;
    return p;
}

// ---- K2: fused decompression + exact MaxSim ---------------------------------------------
template <int NB>
__global__ void __launch_bounds__(kFusedThreads)
stream_fused_kernel(const float* __restrict__ C, const uint32_t* __restrict__ codes,
                    const uint8_t* __restrict__ residuals, Weights16 W, const uint64_t* __restrict__ d_n,
                    const uint32_t* __restrict__ pref, const uint64_t* __restrict__ fin_base,
                    const float* __restrict__ Q, uint32_t rows, uint32_t* __restrict__ run, uint32_t dbg) {
    dev::pdl_wait();
    extern __shared__ __align__(16) float sm[];
    __shared__ float w_s[16];
    // the 4 bucket weights of every (4 NB)-bit residual group (NB <= 2): one
    // LDS.128 per 4 dims instead of 4 index extractions and 4 lookups
    constexpr uint32_t kLutN = NB <= 2 ? (1u << (4 * NB)) : 1u;
    __shared__ float4 w_lut[kLutN];
    __shared__ uint32_t pass_s[2][kTile];
    __shared__ __align__(8) uint64_t full_bar[2], empty_bar[2];
    constexpr uint32_t kBpt = NB * 128 / 8;
    // query pairs interleaved: qp[g][d] = (q_{2g}[d], q_{2g+1}[d]), so one
    // FMUL2 forms both products of a token dim with a query pair
    float2* qp = reinterpret_cast<float2*>(sm);  // 16 x 128 float2
    float* tiles = sm + 16 * 128 * 2;            // 2 x kTile x kPitch
    const uint32_t lane = dev::lane_id(), warp = threadIdx.x >> 5;
    const uint32_t n = uint32_t(*d_n);
    const uint32_t T = pref[n];
    const uint32_t ntiles = (T + kTile - 1) / kTile;
    if (blockIdx.x >= ntiles) return;
    if (threadIdx.x < 16) w_s[threadIdx.x] = W.w[threadIdx.x];
    if (NB <= 2) {
        constexpr uint32_t m = (1u << NB) - 1;
        for (uint32_t e = threadIdx.x; e < kLutN; e += blockDim.x)
            w_lut[e] = make_float4(W.w[e & m], W.w[(e >> NB) & m], W.w[(e >> (2 * NB)) & m], W.w[(e >> (3 * NB)) & m]);
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full_bar[b], kProducers * 32);
            mbar_init(&empty_bar[b], kConsumers * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t i = threadIdx.x; i < 16 * 32; i += kFusedThreads) {
        const uint32_t g = i >> 5, d4 = i & 31;
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 x = 2 * g < rows ? __ldg(reinterpret_cast<const float4*>(Q + 2 * g * 128) + d4) : z;
        const float4 y = 2 * g + 1 < rows ? __ldg(reinterpret_cast<const float4*>(Q + (2 * g + 1) * 128) + d4) : z;
        float4* dst = reinterpret_cast<float4*>(qp + g * 128 + 4 * d4);
        dst[0] = make_float4(x.x, y.x, x.y, y.y);
        dst[1] = make_float4(x.z, y.z, x.w, y.w);
    }
    __syncthreads();

    if (warp >= kConsumers) {
        // ---------------- producers: decompress tiles into the ring
        const uint32_t pw = warp - kConsumers;  // tokens [32 pw, 32 pw + 32) of each tile
        constexpr uint32_t mask = (1u << NB) - 1;
        uint32_t k = 0;
        for (uint32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++k) {
            const uint32_t b = k & 1;
            mbar_wait(&empty_bar[b], ((k >> 1) & 1) ^ 1);
            if (pw == 0) rank_stamp(dbg, 0, k);
            if (dbg & 2) {  // experiment: no decompression (consumers score stale tiles)
                if (k < 2) pass_s[b][pw * 32 + lane] = 0xFFFFFFFFu - pw;
                mbar_arrive(&full_bar[b]);
                continue;
            }
            float* tile = tiles + b * kTile * kPitch + pw * 32 * kPitch;
            const uint32_t g0 = tl * kTile + pw * 32;
            const uint32_t g = g0 + lane;
            const bool valid = g < T;
            uint64_t tok = 0;
            uint32_t code = 0, p = 0xFFFFFFFFu;
            if (g0 < T) p = run_finalists(pref, n, g0, g);
            if (valid) {
                tok = fin_base[p] + g;
                code = __ldg(codes + tok);
            } else {
                p = 0xFFFFFFFFu - pw;  // never equal to a real finalist or to the other half's pad
            }
            pass_s[b][pw * 32 + lane] = p;
            const uint32_t nv = g0 < T ? (T - g0 < 32 ? T - g0 : 32) : 0;
            for (uint32_t t = 0; t < nv; ++t) {
                const uint32_t ct = __shfl_sync(0xffffffffu, code, t);
                cp_async16(tile + t * kPitch + 4 * lane, C + uint64_t(ct) * 128 + 4 * lane);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            uint32_t rb[kBpt / 4];
            if (valid) {
                const uint4* src = reinterpret_cast<const uint4*>(residuals + tok * kBpt);
#pragma unroll
                for (uint32_t i = 0; i < kBpt / 16; ++i) {
                    const uint4 x = __ldg(src + i);
                    rb[4 * i] = x.x, rb[4 * i + 1] = x.y, rb[4 * i + 2] = x.z, rb[4 * i + 3] = x.w;
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            if (pw == 0) rank_stamp(dbg, 1, k);
            if (valid) {
                float4* row = reinterpret_cast<float4*>(tile + lane * kPitch);
                double acc = 0.0;
#pragma unroll
                for (int d4 = 0; d4 < 32; ++d4) {
                    // dims 4*d4 .. 4*d4+3 <- 4*NB bits from bit 4*d4*NB (LSB-first packing)
                    const uint32_t word = rb[(4 * d4 * NB) / 32] >> ((4 * d4 * NB) % 32);
                    float4 x = row[d4];
                    if (NB <= 2) {
                        const float4 w4 = w_lut[word & (kLutN - 1)];
                        x.x = __fadd_rn(x.x, w4.x);
                        x.y = __fadd_rn(x.y, w4.y);
                        x.z = __fadd_rn(x.z, w4.z);
                        x.w = __fadd_rn(x.w, w4.w);
                    } else {
                        x.x = __fadd_rn(x.x, w_s[(word >> (0 * NB)) & mask]);
                        x.y = __fadd_rn(x.y, w_s[(word >> (1 * NB)) & mask]);
                        x.z = __fadd_rn(x.z, w_s[(word >> (2 * NB)) & mask]);
                        x.w = __fadd_rn(x.w, w_s[(word >> (3 * NB)) & mask]);
                    }
                    row[d4] = x;
                    // norm^2 += double(x)^2 in order (residual_codec.cpp:113-130): the
                    // square of a float is exact in double (48 <= 53 significand bits),
                    // so one fused multiply-add rounds exactly like the separate add
                    acc = __fma_rn(double(x.x), double(x.x), acc);
                    acc = __fma_rn(double(x.y), double(x.y), acc);
                    acc = __fma_rn(double(x.z), double(x.z), acc);
                    acc = __fma_rn(double(x.w), double(x.w), acc);
                }
                if (acc > 0.0) {
                    const float inv = float(1.0 / sqrt(acc));
#pragma unroll
                    for (int d4 = 0; d4 < 32; ++d4) {
                        float4 x = row[d4];
                        x.x = __fmul_rn(x.x, inv), x.y = __fmul_rn(x.y, inv);
                        x.z = __fmul_rn(x.z, inv), x.w = __fmul_rn(x.w, inv);
                        row[d4] = x;
                    }
                }
            }
            if (pw == 0) rank_stamp(dbg, 2, k);
            mbar_arrive(&full_bar[b]);
        }
        return;
    }

    // ---------------- consumers: exact MaxSim over ready tiles
    const uint32_t i0 = warp * 8;
    const float4* q4 = reinterpret_cast<const float4*>(qp + (i0 / 2) * 128);
    uint32_t k = 0;
    for (uint32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++k) {
        const uint32_t b = k & 1;
        mbar_wait(&full_bar[b], (k >> 1) & 1);
        if (warp == 0) rank_stamp(dbg, 3, k);
        const float* tile = tiles + b * kTile * kPitch;
        const uint32_t p0 = pass_s[b][lane], p1 = pass_s[b][32 + lane];
        const bool valid0 = p0 < 0xFFFFFFF0u, valid1 = p1 < 0xFFFFFFF0u;
        if (i0 < rows) {
            float a[8], c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = 0.0f, c[u] = 0.0f;
            const float4* vr0 = reinterpret_cast<const float4*>(tile + lane * kPitch);
            const float4* vr1 = reinterpret_cast<const float4*>(tile + (32 + lane) * kPitch);
#pragma unroll 2
            for (uint32_t d4 = 0; d4 < 32; ++d4) {
                const float4 v = vr0[d4], w = vr1[d4];
                const float vv[4] = {v.x, v.y, v.z, v.w}, ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int gp = 0; gp < 4; ++gp) {
                    // (q_u, q_u+1) at dims 4*d4 .. 4*d4+3, u = i0 + 2*gp
                    const float4 qa = q4[gp * 64 + 2 * d4], qb = q4[gp * 64 + 2 * d4 + 1];
                    const float2 qq[4] = {make_float2(qa.x, qa.y), make_float2(qa.z, qa.w),
                                          make_float2(qb.x, qb.y), make_float2(qb.z, qb.w)};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        // products rounded once each (FMUL2), then the in-order adds
                        const float2 q0 = dev::mul2_rn(qq[e], vv[e]), q1 = dev::mul2_rn(qq[e], ww[e]);
                        a[2 * gp] = __fadd_rn(a[2 * gp], q0.x);
                        a[2 * gp + 1] = __fadd_rn(a[2 * gp + 1], q0.y);
                        c[2 * gp] = __fadd_rn(c[2 * gp], q1.x);
                        c[2 * gp + 1] = __fadd_rn(c[2 * gp + 1], q1.y);
                    }
                }
            }
            // segmented max over the lanes of each finalist (its lanes are
            // contiguous); the segment's last lane publishes
            const uint32_t pn0 = __shfl_down_sync(0xffffffffu, p0, 1);
            const uint32_t pn1 = __shfl_down_sync(0xffffffffu, p1, 1);
            const bool tail0 = valid0 && (lane == 31 || pn0 != p0);
            const bool tail1 = valid1 && (lane == 31 || pn1 != p1);
            // segment membership of the lane `o` below, per scan step (same for every query)
            uint32_t same0 = 0, same1 = 0;
#pragma unroll
            for (int l = 0, o = 1; l < 5; ++l, o <<= 1) {
                const uint32_t s0 = __shfl_up_sync(0xffffffffu, p0, o);  // every lane takes part
                const uint32_t s1 = __shfl_up_sync(0xffffffffu, p1, o);
                same0 |= uint32_t(lane >= uint32_t(o) && s0 == p0) << l;
                same1 |= uint32_t(lane >= uint32_t(o) && s1 == p1) << l;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float m0 = a[u], m1 = c[u];
#pragma unroll
                for (int l = 0, o = 1; l < 5; ++l, o <<= 1) {
                    const float y0 = __shfl_up_sync(0xffffffffu, m0, o);
                    const float y1 = __shfl_up_sync(0xffffffffu, m1, o);
                    if ((same0 >> l) & 1u) m0 = dev::max_gt(m0, y0);
                    if ((same1 >> l) & 1u) m1 = dev::max_gt(m1, y1);
                }
                if (i0 + u < rows) {
                    if (tail0) atomicMax(run + uint64_t(p0) * 32 + i0 + u, dev::ord_f32(m0));
                    if (tail1) atomicMax(run + uint64_t(p1) * 32 + i0 + u, dev::ord_f32(m1));
                }
            }
        }
        if (warp == 0) rank_stamp(dbg, 4, k);
        mbar_arrive(&empty_bar[b]);
    }
}

// ---- K2'': stage 4 on mma.sync (TENSOR mode), a warp pair per finalist --------------
// s4_mma.cuh's scorer over finalist f's tokens [fin_base[f] + pref[f],
// + pref[f + 1] - pref[f]) (the finalist scan's outputs), the B fragments
// copied from the query image the prologue built, the finalist's key straight
// out — no running-maxima rows, no finalize.  (A CTA per finalist with its tiles dealt over 4 warps, each CTA
// building its own fragments: 17.9 us against 14.3 at cfg2.)
constexpr uint32_t kS4wThreads = 128;
template <int NB>
__global__ void __launch_bounds__(kS4wThreads)
stage4_warp_kernel(const IndexView ix, const float* __restrict__ S, const uint2* __restrict__ qf, uint32_t rows,
                   const uint64_t* __restrict__ d_n, const uint32_t* __restrict__ pref,
                   const uint64_t* __restrict__ fin_base, const uint32_t* __restrict__ ids,
                   const uint64_t* __restrict__ keys, uint64_t* __restrict__ out_keys) {
    dev::pdl_wait();
    __shared__ uint32_t lut[2 * 256];
    __shared__ float mrows[kS4wThreads];
    __shared__ __align__(16) uint2 qs[s4mma::kQFragBytes / 8];
    constexpr uint32_t kPairs = 1u << (2 * NB), kMask = (1u << NB) - 1;
    for (uint32_t e = threadIdx.x; e < kPairs; e += kS4wThreads) {
        const float w0 = ix.weights[e & kMask], w1 = ix.weights[e >> NB];
        lut[e] = s4mma::bf16_pair(w0, w1);
        lut[256 + e] = s4mma::bf16_pair_lo(w0, w1);
    }
    // the fragments into shared memory: one coalesced round of 16-byte loads
    // (read from global inside the MMA loop they cost 14 -> 16 us)
#pragma unroll
    for (uint32_t u = 0; u < s4mma::kQFragBytes / 16 / kS4wThreads; ++u) {
        const uint32_t e = u * kS4wThreads + threadIdx.x;
        reinterpret_cast<uint4*>(qs)[e] = __ldg(reinterpret_cast<const uint4*>(qf) + e);
    }
    __syncthreads();
    // two warps per finalist (tiles alternate between them, the maxima meet
    // in shared memory): a finalist is ~5 tiles, and one warp chained them
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pair = warp >> 1, sub = warp & 1;
    constexpr uint32_t kPairs2 = kS4wThreads / 64;
    float* mrow = mrows + warp * 32;
    const uint32_t n = uint32_t(*d_n);
    for (uint32_t f0 = blockIdx.x * kPairs2; f0 < n; f0 += gridDim.x * kPairs2) {
        const uint32_t f = f0 + pair;
        if (f < n) {
            const uint32_t p0 = __ldcg(pref + f), p1 = __ldcg(pref + f + 1);
            const uint64_t off = __ldcg(fin_base + f) + p0;
            s4mma::finalist_max<NB>(ix, S, off, p1 - p0, 16 * sub, 32, qs, lut, mrow);
        }
        __syncthreads();
        if (f < n && sub == 0) {
            mrow[lane] = fmaxf(mrow[lane], mrow[32 + lane]);
            __syncwarp();
            if (lane == 0) {
                float total = 0.0f;
                for (uint32_t i = 0; i < rows; ++i) total = __fadd_rn(total, mrow[i]);
                out_keys[f] = dev::make_key(total, finalist_pid(ids, keys, f));
            }
        }
        __syncthreads();  // the pair's rows are rewritten next round
    }
}

// ---- K3: per-finalist score ---------------------------------------------------------
__global__ void finalize_kernel(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ keys,
                                const uint64_t* __restrict__ d_n, uint32_t rows, uint32_t* __restrict__ run,
                                uint64_t* __restrict__ out_keys) {
    dev::pdl_wait();
    const uint64_t n = *d_n;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
        uint4* r4 = reinterpret_cast<uint4*>(run + p * 32);
        uint32_t v[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 x = r4[j];
            v[4 * j] = x.x, v[4 * j + 1] = x.y, v[4 * j + 2] = x.z, v[4 * j + 3] = x.w;
            r4[j] = make_uint4(0, 0, 0, 0);
        }
        float total = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (uint32_t(i) < rows) total = __fadd_rn(total, dev::unord_f32(v[i]));
        out_keys[p] = dev::make_key(total, finalist_pid(ids, keys, p));
    }
}

// ---- K2': stage 4 on the tensor cores (PLAID_SCORES_TENSOR) ----------------------------
// q_i . v_hat_t with v_t = C[c_t] + r_t (residual_codec.cpp:97-132) is
//   (q_i . C[c_t] + q_i . r_t) * inv_t = (S[c_t][i] + (R Q^T)[t][i]) * inv_t,
// where S is this query's S_cq table (3xTF32, |err| < 5e-6, already in L2
// after stage 1), inv_t = 1 / ||v_t|| is computed per token at index load
// (token_inv_kernel: the reference's in-order fp64 norm), and only R Q^T —
// the residual part, rows of 2^b distinct weights — is a GEMM: 128 finalist
// tokens x 32 query tokens per tile on tcgen05 (kind::f16, split bf16,
// R = R_hi + R_lo, Q = Q_hi + Q_lo, three products kept: ~2^-16 relative).
// A token costs 4 B code + 16 b B residuals + 4 B inv_t from HBM and one
// 128-B S row from L2: the 512-B centroid row of the exact path is never read.
//   warps 0-3  token group, thread = token = TMEM lane (warp w owns lanes
//              32w..32w+31).  The metadata of the CTA's next two tiles is
//              prefetched into registers (finalist via run_p0 and one fused
//              (end, fin_base) load, then code, inv_t and the residual words
//              in flight together); per tile: cp.async of the S rows of this
//              and the next tile, residual decode into packed bf16 pairs
//              (LUT), tcgen05.st of A = [R_hi | R_lo] (K = 256, 128 columns);
//              then the epilogue: tcgen05.ld of D, a 32x32 transpose through
//              shared memory, lane = query token: (S + D) * inv over the
//              warp's 32 tokens, fully unrolled with the finalist segments
//              known up front (ballots), one 128-byte row of atomicMax per
//              segment end (warp-uniform).
//   warp 4     TMEM allocation, the B operand (the query image built by
//              query_prologue, one 32 KB bulk copy) and the MMA issuer:
//              16 x (M=128, N=64, K=16): D[:, i] + D[:, 32 + i] =
//              [R_hi | R_lo] . [Q_hi | Q_hi] + [R_hi | R_lo] . [Q_lo | 0].
// Two CTAs per SM (256 TMEM columns each); tiles round-robin over the grid.
constexpr uint32_t kTcTile = 128;
constexpr uint32_t kTcThreads = 160;
constexpr uint32_t kTcTmemCols = 256;
constexpr uint32_t kTcAccCol = 128;
constexpr uint32_t kTcOffB = 0;                                   // query image (launch::kQImgBytes)
constexpr uint32_t kTcSPitch = 36;                                // floats per S row slot (conflict-free LDS.128)
constexpr uint32_t kTcOffS = kTcOffB + launch::kQImgBytes;        // 2 x 128 tokens x 36 floats
constexpr uint32_t kTcOffTr = kTcOffS + 2 * kTcTile * kTcSPitch * 4;  // 4 warps x 32 x 33 floats
constexpr uint32_t kTcOffLut = kTcOffTr + 4 * 32 * 33 * 4;        // hi[256], lo[256] u32
constexpr uint32_t kTcOffBar = kTcOffLut + 2 * 256 * 4;           // b_full, a_full, acc_full, tmem slot
constexpr uint32_t kTcSmemBytes = kTcOffBar + 64 + 1024;          // + alignment slack
static_assert(2 * (kTcSmemBytes + 1024) <= 228 * 1024, "two CTAs per SM");

// kind::f16 instruction descriptor: D f32, A and B bf16, both K-major, M = 128, N = 64.
constexpr uint32_t kTcIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint64_t tc_desc(uint32_t addr) {
    uint64_t d = uint64_t((addr >> 4) & 0x3FFFu);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

__device__ __forceinline__ void tc_mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void tc_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint16_t bf16_rn_bits(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float bf16_val(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }

__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// Debug timeline (plaid_debug_s4_set(1)): globaltimer stamps per CTA (< 512):
// 0 start, 1 prefetch done, 2 B landed (MMA warp), 3/6/9 tile 0/1/2 A stored,
// 4/7/10 D ready, 5/8/11 epilogue done, 12 end (token warp 0, lane 0).
__device__ unsigned long long g_s4_trace[512 * 16];
__device__ uint32_t g_s4_dbg;
__device__ __forceinline__ void s4_stamp(int ev) {
    if (g_s4_dbg && blockIdx.x < 512 && (threadIdx.x & 31) == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_s4_trace[blockIdx.x * 16 + ev] = t;
    }
}

// One lane's token of a tile: what the decode and the epilogue need, loaded
// ahead of use (residual words, code, inv_t in flight).
template <int NB>
struct TcToken {
    uint32_t rb[NB * 128 / 32];
    uint32_t code;
    float inv;
    uint32_t p;  // finalist index, 0xFFFFFFFF past the stream end
};

// Finalists of the warp's 32-token run [g0, g0 + 32) of tile `tl` (g0 < T):
// first the run's first finalist lo (run_p0), then lane j loads the end of
// finalist lo + j and its token base in ONE step; the finalist of lane L is
// lo + #{j : end_j <= g0 + L} (ends are distinct: each finalist has a token).
template <int NB>
__device__ __forceinline__ void tc_prefetch2(TcToken<NB>& a, TcToken<NB>& b, uint32_t tla, uint32_t tlb, uint32_t ntiles,
                                             uint32_t T, uint32_t n, const uint32_t* __restrict__ pref,
                                             const uint64_t* __restrict__ fin_base,
                                             const uint32_t* __restrict__ run_p0, const uint32_t* __restrict__ codes,
                                             const float* __restrict__ tok_inv, const uint8_t* __restrict__ residuals) {
    constexpr uint32_t kBpt = NB * 128 / 8;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g0a = tla * kTcTile + warp * 32, g0b = tlb * kTcTile + warp * 32;
    const bool ha = tla < ntiles && g0a < T, hb = tlb < ntiles && g0b < T;
    const uint32_t loa = ha ? __ldg(run_p0 + (g0a >> 5)) : 0u;
    const uint32_t lob = hb ? __ldg(run_p0 + (g0b >> 5)) : 0u;
    const bool ia = ha && loa + 1 + lane <= n, ib = hb && lob + 1 + lane <= n;
    const uint32_t ea = ia ? __ldg(pref + loa + 1 + lane) : 0xFFFFFFFFu;
    const uint32_t eb = ib ? __ldg(pref + lob + 1 + lane) : 0xFFFFFFFFu;
    const uint64_t fa = ia ? __ldg(reinterpret_cast<const unsigned long long*>(fin_base) + loa + lane) : 0ull;
    const uint64_t fb = ib ? __ldg(reinterpret_cast<const unsigned long long*>(fin_base) + lob + lane) : 0ull;
    auto finish = [&](TcToken<NB>& x, bool has, uint32_t g0, uint32_t lo, uint32_t e, uint64_t f) {
        const uint32_t rel = e - g0;  // > 0: finalist lo holds g0
        const uint32_t mask = __reduce_or_sync(0xffffffffu, has && rel < 32 ? 1u << rel : 0u);
        const uint32_t cnt = __popc(mask & (0xFFFFFFFFu >> (31 - lane)));  // ends at or before g0 + lane
        const uint64_t base = __shfl_sync(0xffffffffu, f, cnt);
        const uint32_t g = g0 + lane;
        if (has && g < T) {
            x.p = lo + cnt;
            const uint64_t tok = base + g;
            x.code = __ldg(codes + tok);
            x.inv = __ldg(tok_inv + tok);
            const uint4* src = reinterpret_cast<const uint4*>(residuals + tok * kBpt);
#pragma unroll
            for (uint32_t i = 0; i < kBpt / 16; ++i) {
                const uint4 v = __ldg(src + i);
                x.rb[4 * i] = v.x, x.rb[4 * i + 1] = v.y, x.rb[4 * i + 2] = v.z, x.rb[4 * i + 3] = v.w;
            }
        } else {
            x.p = 0xFFFFFFFFu;
            x.code = 0u;
            x.inv = 0.0f;
#pragma unroll
            for (uint32_t i = 0; i < kBpt / 4; ++i) x.rb[i] = 0u;
        }
    };
    finish(a, ha, g0a, loa, ea, fa);
    finish(b, hb, g0b, lob, eb, fb);
}

// cp.async of the token's 128-byte S row into its row of an S slot (skipped
// past the stream end); one commit group per call
template <int NB>
__device__ __forceinline__ void tc_fetch_srow(const TcToken<NB>& x, const float* __restrict__ S, float* srow_slot) {
    if (x.p != 0xFFFFFFFFu) {
        const float* src = S + uint64_t(x.code) * kScoresPitch;
        float* dst = srow_slot + threadIdx.x * kTcSPitch;
#pragma unroll
        for (int c = 0; c < 8; ++c) cp_async16(dst + 4 * c, src + 4 * c);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// A operand of the token's TMEM lane: columns [0, 64) packed bf16 pairs of
// R_hi, [64, 128) of R_lo; then the warp's arrival on a_full
template <int NB>
__device__ __forceinline__ void tc_store_a(const TcToken<NB>& x, uint32_t tmem, uint32_t a_full,
                                           const uint32_t* lut_hi, const uint32_t* lut_lo) {
    constexpr uint32_t kPairBits = 2 * NB, kPairs = 1u << kPairBits;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lane_off = (warp * 32) << 16;
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (uint32_t c = 0; c < 32; ++c) {
            const uint32_t bit = (32 * h + c) * kPairBits;
            const uint32_t e = (x.rb[bit / 32] >> (bit % 32)) & (kPairs - 1);
            hi[c] = lut_hi[e];
            lo[c] = lut_lo[e];
        }
        tc_st32(tmem + lane_off + 32 * h, hi);
        tc_st32(tmem + lane_off + 64 + 32 * h, lo);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) tc_mbar_arrive(a_full);
}

// D of tile lt into registers: d[i] = D[:, i] + D[:, 32 + i] = q_i . r_t
__device__ __forceinline__ void tc_read_d(uint32_t lt, uint32_t tmem, uint32_t acc_full, float (&d)[32]) {
    const uint32_t warp = threadIdx.x >> 5;
    tc_mbar_wait(acc_full, lt & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t d0[32], d1[32];
    tc_ld32(tmem + ((warp * 32) << 16) + kTcAccCol, d0);
    tc_ld32(tmem + ((warp * 32) << 16) + kTcAccCol + 32, d1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) d[i] = __uint_as_float(d0[i]) + __uint_as_float(d1[i]);
}

// Epilogue of a tile (its S rows landed): thread = token forms the 32 scores
// (S + D) * inv, a transpose through shared memory puts lane = query token,
// and the warp walks its 32 tokens in stream order: the max restarts at a
// finalist's first token and is published (one coalesced 128-byte row of
// atomicMax) at its last — segments known up front from two ballots.
__device__ __forceinline__ void tc_epilogue(float (&d)[32], float inv, uint32_t my_p, const float* srow_slot,
                                            float* tr, uint32_t rows, uint32_t* __restrict__ run) {
    const uint32_t lane = threadIdx.x & 31;
    const float4* s4 = reinterpret_cast<const float4*>(srow_slot + threadIdx.x * kTcSPitch);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float4 sv = s4[c];
        tr[lane * 33 + 4 * c + 0] = __fmul_rn(__fadd_rn(sv.x, d[4 * c + 0]), inv);
        tr[lane * 33 + 4 * c + 1] = __fmul_rn(__fadd_rn(sv.y, d[4 * c + 1]), inv);
        tr[lane * 33 + 4 * c + 2] = __fmul_rn(__fadd_rn(sv.z, d[4 * c + 2]), inv);
        tr[lane * 33 + 4 * c + 3] = __fmul_rn(__fadd_rn(sv.w, d[4 * c + 3]), inv);
    }
    const uint32_t prev_p = __shfl_up_sync(0xffffffffu, my_p, 1), next_p = __shfl_down_sync(0xffffffffu, my_p, 1);
    const bool tok = my_p != 0xFFFFFFFFu;
    const uint32_t starts = __ballot_sync(0xffffffffu, tok && (lane == 0 || prev_p != my_p));
    const uint32_t ends = __ballot_sync(0xffffffffu, tok && (lane == 31 || next_p != my_p));
    __syncwarp();
    const uint32_t i = lane;
    const bool live = i < rows;
    float m = 0.0f;
#pragma unroll
    for (uint32_t t = 0; t < 32; ++t) {
        const float v = tr[t * 33 + i];
        m = ((starts >> t) & 1u) ? v : dev::max_gt(m, v);
        if ((ends >> t) & 1u) {
            const uint32_t pt = __shfl_sync(0xffffffffu, my_p, t);
            if (live) atomicMax(run + uint64_t(pt) * 32 + i, dev::ord_f32(m));
        }
    }
    __syncwarp();
}

template <int NB>
__global__ void __launch_bounds__(kTcThreads, 2)
stage4_tensor_kernel(const float* __restrict__ S, const float* __restrict__ tok_inv, const uint32_t* __restrict__ codes,
                     const uint8_t* __restrict__ residuals, Weights16 W, const uint64_t* __restrict__ d_n,
                     const uint32_t* __restrict__ pref, const uint64_t* __restrict__ fin_base,
                     const uint32_t* __restrict__ run_p0, const uint8_t* __restrict__ qimg, uint32_t rows,
                     uint32_t* __restrict__ run) {
    dev::pdl_wait();
    extern __shared__ __align__(16) uint8_t tc_smem_raw[];
    uint8_t* smem = tc_smem_raw + ((1024u - (smem_addr(tc_smem_raw) & 1023u)) & 1023u);
    const uint32_t base = smem_addr(smem);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t b_full = base + kTcOffBar, a_full = base + kTcOffBar + 8, acc_full = base + kTcOffBar + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kTcOffBar + 24);
    float* srow = reinterpret_cast<float*>(smem + kTcOffS);
    float* trb = reinterpret_cast<float*>(smem + kTcOffTr);
    uint32_t* lut_hi = reinterpret_cast<uint32_t*>(smem + kTcOffLut);
    uint32_t* lut_lo = lut_hi + 256;

    const uint32_t n = uint32_t(*d_n);
    const uint32_t T = pref[n];
    const uint32_t ntiles = (T + kTcTile - 1) / kTcTile;
    if (blockIdx.x >= ntiles) return;
    if (warp == 0) s4_stamp(0);

    // LUT: a residual bit group of two dims (2 NB bits, LSB first) -> packed
    // bf16 pairs (low half = the even dim) of w_hi and of w_lo = w - w_hi
    constexpr uint32_t kPairs = 1u << (2 * NB), kMask = (1u << NB) - 1;
    for (uint32_t e = threadIdx.x; e < kPairs; e += kTcThreads) {
        const float wa = W.w[e & kMask], wb = W.w[(e >> NB) & kMask];
        const uint16_t ha = bf16_rn_bits(wa), hb = bf16_rn_bits(wb);
        const uint16_t la = bf16_rn_bits(wa - bf16_val(ha)), lb = bf16_rn_bits(wb - bf16_val(hb));
        lut_hi[e] = uint32_t(ha) | (uint32_t(hb) << 16);
        lut_lo[e] = uint32_t(la) | (uint32_t(lb) << 16);
    }
    if (threadIdx.x == 0) {
        tc_mbar_init(b_full, 1);
        tc_mbar_init(a_full, 4);
        tc_mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(kTcTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        // ---------------- B operand + MMA issuer
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b_full), "r"(launch::kQImgBytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    base + kTcOffB),
                "l"(qimg), "r"(launch::kQImgBytes), "r"(b_full)
                : "memory");
        }
        tc_mbar_wait(b_full, 0);
        s4_stamp(2);
        uint32_t lt = 0;
        for (uint32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++lt) {
            tc_mbar_wait(a_full, lt & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // D[:, 0:32] = [R_hi | R_lo] . [Q_hi | Q_hi], D[:, 32:64] = [R_hi | R_lo] . [Q_lo | 0]:
            // 16 K=16 steps (B chunk s >> 2, 32-byte step s & 3: +512 / +2 in the
            // descriptor's address field; A +8 TMEM columns), issued by the
            // converged warp with the elected lane predicated inside one asm
            // block (no per-MMA waterfall loop, see gemm_tf32.cu mma_chunk_tf32)
            asm volatile(
                "{\n\t"
                ".reg .pred e, pz, pt;\n\t"
                ".reg .b32 rx, ta;\n\t"
                ".reg .b64 bd;\n\t"
                "elect.sync rx|e, 0xffffffff;\n\t"
                "setp.ne.b32 pz, %1, %1;\n\t"
                "setp.eq.b32 pt, %1, %1;\n\t"
                "add.s64 bd, %2, 0;\n\t"
                "add.u32 ta, %1, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pz;\n\t"
                "add.s64 bd, %2, 2;\n\t"
                "add.u32 ta, %1, 8;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 4;\n\t"
                "add.u32 ta, %1, 16;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 6;\n\t"
                "add.u32 ta, %1, 24;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 512;\n\t"
                "add.u32 ta, %1, 32;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 514;\n\t"
                "add.u32 ta, %1, 40;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 516;\n\t"
                "add.u32 ta, %1, 48;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 518;\n\t"
                "add.u32 ta, %1, 56;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1024;\n\t"
                "add.u32 ta, %1, 64;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1026;\n\t"
                "add.u32 ta, %1, 72;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1028;\n\t"
                "add.u32 ta, %1, 80;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1030;\n\t"
                "add.u32 ta, %1, 88;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1536;\n\t"
                "add.u32 ta, %1, 96;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1538;\n\t"
                "add.u32 ta, %1, 104;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1540;\n\t"
                "add.u32 ta, %1, 112;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "add.s64 bd, %2, 1542;\n\t"
                "add.u32 ta, %1, 120;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, pt;\n\t"
                "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t"
                "}" ::"r"(tmem + kTcAccCol),
                "r"(tmem), "l"(tc_desc(base + kTcOffB)), "r"(kTcIdesc), "r"(acc_full)
                : "memory");
        }
    } else {
        // ---------------- token group: a two-stage software pipeline — while
        // tile lt's epilogue runs, tile lt + 1's A operand is in TMEM and its
        // MMAs are in flight
        float* tr = trb + warp * 32 * 33;
        TcToken<NB> x0, x1;
        const uint32_t G = gridDim.x;
        tc_prefetch2<NB>(x0, x1, blockIdx.x, blockIdx.x + G, ntiles, T, n, pref, fin_base, run_p0, codes, tok_inv,
                         residuals);
        if (warp == 0) s4_stamp(1);
        float* srow1 = srow + kTcTile * kTcSPitch;
        tc_store_a<NB>(x0, tmem, a_full, lut_hi, lut_lo);
        if (warp == 0) s4_stamp(3);
        tc_fetch_srow<NB>(x0, S, srow);
        float d[32];
        TcToken<NB> unused;
        uint32_t lt = 0;
        for (uint32_t tl = blockIdx.x; tl < ntiles; tl += 2 * G, lt += 2) {
            // tile lt: metadata x0, S slot 0; tile lt + 1: x1, slot 1; the
            // metadata of tile lt + 2 is requested before tile lt's epilogue
            const bool has1 = tl + G < ntiles, has2 = tl + 2 * G < ntiles;
            tc_read_d(lt, tmem, acc_full, d);
            if (warp == 0 && lt < 3) s4_stamp(4 + 3 * lt);
            if (has1) {
                tc_store_a<NB>(x1, tmem, a_full, lut_hi, lut_lo);
                if (warp == 0 && lt + 1 < 3) s4_stamp(3 + 3 * (lt + 1));
                tc_fetch_srow<NB>(x1, S, srow1);
            }
            float inv = x0.inv;
            uint32_t pp = x0.p;
            if (has2)
                tc_prefetch2<NB>(x0, unused, tl + 2 * G, ntiles, ntiles, T, n, pref, fin_base, run_p0, codes, tok_inv,
                                 residuals);
            if (has1)
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            else
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            tc_epilogue(d, inv, pp, srow, tr, rows, run);
            if (warp == 0 && lt < 3) s4_stamp(5 + 3 * lt);
            if (!has1) break;
            // tile lt + 1 (x1, slot 1); tile lt + 2 (x0, slot 0) goes to TMEM
            const bool has3 = tl + 3 * G < ntiles;
            tc_read_d(lt + 1, tmem, acc_full, d);
            if (warp == 0 && lt + 1 < 3) s4_stamp(4 + 3 * (lt + 1));
            if (has2) {
                tc_store_a<NB>(x0, tmem, a_full, lut_hi, lut_lo);
                if (warp == 0 && lt + 2 < 3) s4_stamp(3 + 3 * (lt + 2));
                tc_fetch_srow<NB>(x0, S, srow);
            }
            inv = x1.inv;
            pp = x1.p;
            if (has3)
                tc_prefetch2<NB>(x1, unused, tl + 3 * G, ntiles, ntiles, T, n, pref, fin_base, run_p0, codes, tok_inv,
                                 residuals);
            if (has2)
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            else
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            tc_epilogue(d, inv, pp, srow1, tr, rows, run);
            if (warp == 0 && lt + 1 < 3) s4_stamp(5 + 3 * (lt + 1));
            if (!has2) break;
        }
    }
    if (warp == 0) s4_stamp(12);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 4)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmemCols));
}

// inv_t = 1 / ||C[c_t] + w[idx_t]|| per index token, with the reference's
// arithmetic (residual_codec.cpp:113-130: fp32 adds, in-order fp64 norm,
// float(1 / sqrt)); 1 for a zero vector (the reference leaves it unscaled).
// Index-load time, one thread per token.
template <int NB>
__global__ void token_inv_kernel(const float* __restrict__ C, const uint32_t* __restrict__ codes,
                                 const uint8_t* __restrict__ residuals, Weights16 W, uint64_t T, uint64_t K,
                                 float* __restrict__ out) {
    constexpr uint32_t kBpt = NB * 128 / 8, kMask = (1u << NB) - 1;
    __shared__ float w_s[16];
    if (threadIdx.x < 16) w_s[threadIdx.x] = W.w[threadIdx.x];
    __syncthreads();
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < T; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t code = __ldg(codes + t);
        if (code >= K) {  // not yet validated (an on-disk index is checksummed after upload)
            out[t] = 0.0f;
            continue;
        }
        const float4* c4 = reinterpret_cast<const float4*>(C + uint64_t(code) * 128);
        uint32_t rb[kBpt / 4];
        const uint4* src = reinterpret_cast<const uint4*>(residuals + t * kBpt);
#pragma unroll
        for (uint32_t i = 0; i < kBpt / 16; ++i) {
            const uint4 x = __ldg(src + i);
            rb[4 * i] = x.x, rb[4 * i + 1] = x.y, rb[4 * i + 2] = x.z, rb[4 * i + 3] = x.w;
        }
        double acc = 0.0;
#pragma unroll 8
        for (uint32_t d4 = 0; d4 < 32; ++d4) {
            const float4 c = __ldg(c4 + d4);
            const float cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t d = 4 * d4 + u, bit = d * NB;
                const float v = __fadd_rn(cc[u], w_s[(rb[bit / 32] >> (bit % 32)) & kMask]);
                acc = __fma_rn(double(v), double(v), acc);  // exact square + one rounding = the in-order add
            }
        }
        out[t] = acc > 0.0 ? float(1.0 / sqrt(acc)) : 1.0f;
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

bool rank_stream128_ok(const IndexView& ix, uint32_t rows, uint64_t nmax, const RankScratch& s) {
    return ix.dim == 128 && rows <= 32 && nmax <= s.pass_cap && nmax * ix.max_doclen < (1ull << 32);
}

bool rank_stream128(const IndexView& ix, const float* d_q, uint32_t rows, const uint32_t* d_ids,
                    const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t* d_out_keys,
                    const RankScratch& s, cudaStream_t st) {
    if (!rank_stream128_ok(ix, rows, nmax, s)) return false;
    Weights16 W;
    for (int i = 0; i < 16; ++i) W.w[i] = ix.weights[i];
    const size_t fsm = size_t(kSmemFloats) * sizeof(float);
    static launch::PerDeviceOnce cfg;
    if (cfg.first()) {
        cudaFuncSetAttribute(stream_fused_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fsm));
        cudaFuncSetAttribute(stream_fused_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fsm));
        cudaFuncSetAttribute(stream_fused_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fsm));
    }
    if (!s.prescanned) {
        ::plaid::launch::pdl(finalist_scan_kernel, 1, 1024, 0, st, d_ids, d_keys, d_n, ix.doclens, ix.offsets, s.pref,
                             s.fin_base, s.tokens, s.tensor_S ? s.run_p0 : static_cast<uint32_t*>(nullptr));
        count_launch();
    }
    if (s.tensor_S && ix.tok_inv && s.warp_s4 && s.qimg) {
        // TENSOR mode, a warp per finalist: keys straight out (no finalize)
        const uint32_t per_cta = kS4wThreads / 64;  // finalists per CTA (two warps each)
        const uint32_t blocks = uint32_t(std::max<uint64_t>(1, (nmax + per_cta - 1) / per_cta));
        auto wk = ix.nbits == 1 ? stage4_warp_kernel<1> : ix.nbits == 2 ? stage4_warp_kernel<2> : stage4_warp_kernel<4>;
        const uint2* qf = reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(s.qimg) + kQImgBytes);
        ::plaid::launch::pdl(wk, blocks, kS4wThreads, 0, st, ix, s.tensor_S, qf, rows, d_n, s.pref, s.fin_base,
                             d_ids, d_keys, d_out_keys);
        count_launch();
        return true;
    }
    uint64_t fb = (nmax * ix.max_doclen + kTile - 1) / kTile;
    if (fb > uint64_t(sm_count()) * 2) fb = uint64_t(sm_count()) * 2;  // two CTAs (12 warps) per SM
    if (s.tensor_S && ix.tok_inv && s.run_p0 && s.qimg) {
        // TENSOR mode: residual products on tcgen05, S rows reused (stage4_tensor_kernel)
        static launch::PerDeviceOnce tcfg;
        if (tcfg.first()) {
            cudaFuncSetAttribute(stage4_tensor_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmemBytes));
            cudaFuncSetAttribute(stage4_tensor_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmemBytes));
            cudaFuncSetAttribute(stage4_tensor_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmemBytes));
        }
        uint64_t tb = (nmax * ix.max_doclen + kTcTile - 1) / kTcTile;
        if (tb > uint64_t(sm_count()) * 2) tb = uint64_t(sm_count()) * 2;  // two CTAs (2 x 256 TMEM columns) per SM
        if (tb == 0) tb = 1;
        auto tk = ix.nbits == 1 ? stage4_tensor_kernel<1> : ix.nbits == 2 ? stage4_tensor_kernel<2> : stage4_tensor_kernel<4>;
        ::plaid::launch::pdl(tk, uint32_t(tb), kTcThreads, kTcSmemBytes, st, s.tensor_S, ix.tok_inv, ix.codes,
                             ix.residuals, W, d_n, s.pref, s.fin_base, s.run_p0,
                             static_cast<const uint8_t*>(s.qimg), rows, s.run);
        count_launch();
    } else {
        auto fk = ix.nbits == 1 ? stream_fused_kernel<1> : ix.nbits == 2 ? stream_fused_kernel<2> : stream_fused_kernel<4>;
        static const uint32_t dbg = [] {
            const char* e = getenv("PLAID_RANK_DBG");
            return e ? uint32_t(atoi(e)) : 0u;
        }();
        ::plaid::launch::pdl(fk, uint32_t(fb), kFusedThreads, fsm, st, ix.centroids, ix.codes, ix.residuals, W, d_n, s.pref,
                             s.fin_base, d_q, rows, s.run, dbg);
        count_launch();
    }
    if (s.final_out) {  // finalize + top-k sort in one launch
        const RankScratch::Final& f = *s.final_out;
        finalize_rank(d_ids, d_keys, d_n, nmax, rows, s.run, f.want, f.ids, f.scores, f.n, f.base, f.ticket, st);
        return true;
    }
    const uint32_t nb = uint32_t((nmax + 255) / 256);
    ::plaid::launch::pdl(finalize_kernel, nb, 256, 0, st, d_ids, d_keys, d_n, rows, s.run, d_out_keys);
    count_launch();
    return true;
}

void token_inv_norms(const IndexView& ix, float* d_out, cudaStream_t st) {
    if (ix.dim != 128 || ix.T == 0) return;
    Weights16 W;
    for (int i = 0; i < 16; ++i) W.w[i] = ix.weights[i];
    const uint64_t blocks = std::min<uint64_t>((ix.T + 255) / 256, uint64_t(sm_count()) * 16);
    auto k = ix.nbits == 1 ? token_inv_kernel<1> : ix.nbits == 2 ? token_inv_kernel<2> : token_inv_kernel<4>;
    k<<<uint32_t(blocks), 256, 0, st>>>(ix.centroids, ix.codes, ix.residuals, W, ix.T, ix.K, d_out);
    count_launch();
}

}  // namespace launch
}  // namespace plaid

// Debug: CTA 0's stage-4 tile timeline (see rank_stamp), 5 x 64 stamps.
extern "C" int plaid_debug_rank_trace(unsigned long long* out) {
    return int(cudaMemcpyFromSymbol(out, plaid::g_rank_trace, sizeof(plaid::g_rank_trace)));
}

// Debug: the tensor-core stage-4 timeline (s4_stamp), 512 CTAs x 16 stamps.
extern "C" int plaid_debug_s4_set(uint32_t on) {
    int rc = int(cudaMemcpyToSymbol(plaid::g_s4_dbg, &on, sizeof on));
    unsigned long long z[512 * 16] = {};
    if (!rc) rc = int(cudaMemcpyToSymbol(plaid::g_s4_trace, z, sizeof z));
    return rc;
}
extern "C" int plaid_debug_s4_trace(unsigned long long* out) {
    return int(cudaMemcpyFromSymbol(out, plaid::g_s4_trace, sizeof(plaid::g_s4_trace)));
}
