// s4_mma.cuh — stage 4 in TENSOR score mode on the warp-level tensor path
// (mma.sync), a warp per finalist: used by the throughput worker
// (wave_worker.cu) and by the latency path's stage4_warp_kernel (rank128.cu).
//
// q_i . v_t with v_t = (C[c_t] + r_t) * inv_t (residual_codec.cpp:97-132) is
// computed as (S[c_t][i] + r_t . q_i) * inv_t: S is the query's S_cq table
// (3xTF32), inv_t the per-token norm precomputed at index load
// (token_inv_norms), and only r_t . q_i — rows of 2^NB distinct weights — is
// a GEMM: 16 finalist tokens x 32 query tokens per warp step as m16n8k16 bf16
// MMAs (A = the tokens' residual weights from a LUT of packed bf16 pairs,
// B = Q fragments staged once per CTA), split three ways (R_hi Q_hi + R_hi Q_lo
// + R_lo Q_hi: ~2^-16 relative on the residual term).  MaxSim then takes the
// max over the finalist's tokens (a 16-row reduction across the fragment's
// lane groups) and the in-order fp32 sum over the query tokens
// (maxsim.cpp:66-104).  Scores are within ~1e-6 relative of the exact MaxSim
// (north_star allows 1e-4; oracle/compare.py classifies them).  Device-only.
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"

namespace plaid {
namespace s4mma {

constexpr uint32_t kQFragBytes = 8 * 4 * 2 * 32 * 8;  // [k-step][n-tile][hi, lo][lane] uint2
constexpr uint32_t kLutBytes = 2 * 256 * 4;           // [hi, lo][pair index] u32

// D += A . B, m16n8k16, bf16 in, fp32 accumulate
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// (x, y) -> packed bf16 pair (x in the low half) rounded to nearest, and the
// pair of what rounding left over
__device__ __forceinline__ uint32_t bf16_pair(float x, float y) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(x, y);
    return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t bf16_pair_lo(float x, float y) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    return bf16_pair(x - __low2float(h), y - __high2float(h));
}

// Every thread of the CTA: Q's B fragments (lane ln holds (Q[n][k0],
// Q[n][k0 + 1]) and (Q[n][k0 + 8], Q[n][k0 + 9]), n = 8 j + ln / 4,
// k0 = 16 ks + 2 (ln % 4)) and the residual-pair LUT (index = bucket(d) |
// bucket(d + 1) << NB; dim d's bucket is bits [NB d, NB d + NB) of the
// token's little-endian residual row).  The caller syncs before use.
template <int NB>
__device__ __forceinline__ void setup(const IndexView& ix, const float* __restrict__ Q, uint32_t rows, uint2* qf,
                                      uint32_t* lut) {
    for (uint32_t e = threadIdx.x; e < 8 * 4 * 32; e += blockDim.x) {
        const uint32_t ln = e & 31, j = (e >> 5) & 3, ks = e >> 7;
        const uint32_t n = 8 * j + (ln >> 2), k0 = 16 * ks + 2 * (ln & 3);
        float x[4] = {0.f, 0.f, 0.f, 0.f};
        if (n < rows) {
            const float* qr = Q + uint64_t(n) * 128 + k0;
            x[0] = __ldg(qr), x[1] = __ldg(qr + 1), x[2] = __ldg(qr + 8), x[3] = __ldg(qr + 9);
        }
        qf[((ks * 4 + j) * 2 + 0) * 32 + ln] = make_uint2(bf16_pair(x[0], x[1]), bf16_pair(x[2], x[3]));
        qf[((ks * 4 + j) * 2 + 1) * 32 + ln] = make_uint2(bf16_pair_lo(x[0], x[1]), bf16_pair_lo(x[2], x[3]));
    }
    constexpr uint32_t kPairs = 1u << (2 * NB), kMask = (1u << NB) - 1;
    for (uint32_t e = threadIdx.x; e < kPairs; e += blockDim.x) {
        const float w0 = ix.weights[e & kMask], w1 = ix.weights[e >> NB];
        lut[e] = bf16_pair(w0, w1);
        lut[256 + e] = bf16_pair_lo(w0, w1);
    }
}

// One 16-token tile's loads: rows g (token t0 + g) and g + 8.
template <int NB>
struct Tile {
    uint32_t ca, cb;
    float ia, ib;
    uint32_t ra[NB * 4], rb[NB * 4];
};

template <int NB>
__device__ __forceinline__ void load_tile(const IndexView& ix, uint64_t off, uint32_t len, uint32_t t0, Tile<NB>& d) {
    const uint32_t g = (threadIdx.x & 31) >> 2;
    const uint32_t ta = t0 + g, tb = t0 + g + 8;
    const uint64_t tka = off + (ta < len ? ta : len - 1), tkb = off + (tb < len ? tb : len - 1);
    d.ca = __ldg(ix.codes + tka), d.cb = __ldg(ix.codes + tkb);
    d.ia = __ldg(ix.tok_inv + tka), d.ib = __ldg(ix.tok_inv + tkb);
#pragma unroll
    for (uint32_t x = 0; x < NB * 4; x += 4) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(ix.residuals + tka * (NB * 16)) + x / 4);
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(ix.residuals + tkb * (NB * 16)) + x / 4);
        d.ra[x] = u.x, d.ra[x + 1] = u.y, d.ra[x + 2] = u.z, d.ra[x + 3] = u.w;
        d.rb[x] = v.x, d.rb[x + 1] = v.y, d.rb[x + 2] = v.z, d.rb[x + 3] = v.w;
    }
}

// The warp's per-query-token maxima over tiles t0 = first, first + step, ...
// of finalist (off, len) into mrow[0..32) (-inf without a token).  The next
// tile's codes, norms and residual words are loaded while the current one
// is multiplied.
template <int NB>
__device__ __forceinline__ void finalist_max(const IndexView& ix, const float* __restrict__ S, uint64_t off,
                                             uint32_t len, uint32_t first, uint32_t step, const uint2* qf,
                                             const uint32_t* lut, float* mrow) {
    const uint32_t lane = threadIdx.x & 31, g = lane >> 2, q4 = lane & 3;
    constexpr uint32_t kPairs = 1u << (2 * NB);
    float bm[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) bm[x] = -INFINITY;
    Tile<NB> cur;
    if (first < len) load_tile<NB>(ix, off, len, first, cur);
    for (uint32_t t0 = first; t0 < len; t0 += step) {
        const bool va = t0 + g < len, vb = t0 + g + 8 < len;
        float2 sa[4], sb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sa[j] = __ldg(reinterpret_cast<const float2*>(S + uint64_t(cur.ca) * kScoresPitch + 8 * j + 2 * q4));
            sb[j] = __ldg(reinterpret_cast<const float2*>(S + uint64_t(cur.cb) * kScoresPitch + 8 * j + 2 * q4));
        }
        Tile<NB> nxt;
        if (t0 + step < len) load_tile<NB>(ix, off, len, t0 + step, nxt);
        float acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
        for (uint32_t ks = 0; ks < 8; ++ks) {
            // dims d0 = 16 ks + 2 q4 and d0 + 8: bit NB d0 of the row
            const uint32_t p0 = NB * (16 * ks), sh0 = (p0 & 31) + NB * 2 * q4;
            const uint32_t w0 = p0 >> 5, w1 = (p0 + NB * 8) >> 5, sh1 = ((p0 + NB * 8) & 31) + NB * 2 * q4;
            const uint32_t ia0 = (cur.ra[w0] >> sh0) & (kPairs - 1), ib0 = (cur.rb[w0] >> sh0) & (kPairs - 1);
            const uint32_t ia1 = (cur.ra[w1] >> sh1) & (kPairs - 1), ib1 = (cur.rb[w1] >> sh1) & (kPairs - 1);
            const uint32_t ah[4] = {lut[ia0], lut[ib0], lut[ia1], lut[ib1]};
            const uint32_t al[4] = {lut[256 + ia0], lut[256 + ib0], lut[256 + ia1], lut[256 + ib1]};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint2 bh = qf[((ks * 4 + j) * 2 + 0) * 32 + lane];
                const uint2 bl = qf[((ks * 4 + j) * 2 + 1) * 32 + lane];
                mma_bf16(acc[j], ah, bh.x, bh.y);
                mma_bf16(acc[j], ah, bl.x, bl.y);
                mma_bf16(acc[j], al, bh.x, bh.y);
            }
        }
        // rows g (token t0 + g) and g + 8, columns 8 j + 2 q4 + {0, 1}
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float xa0 = va ? __fmul_rn(__fadd_rn(sa[j].x, acc[j][0]), cur.ia) : -INFINITY;
            const float xa1 = va ? __fmul_rn(__fadd_rn(sa[j].y, acc[j][1]), cur.ia) : -INFINITY;
            const float xb0 = vb ? __fmul_rn(__fadd_rn(sb[j].x, acc[j][2]), cur.ib) : -INFINITY;
            const float xb1 = vb ? __fmul_rn(__fadd_rn(sb[j].y, acc[j][3]), cur.ib) : -INFINITY;
            float m0 = fmaxf(xa0, xb0), m1 = fmaxf(xa1, xb1);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
                m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
            }
            bm[2 * j] = fmaxf(bm[2 * j], m0);
            bm[2 * j + 1] = fmaxf(bm[2 * j + 1], m1);
        }
        cur = nxt;
    }
    // lanes 0-3 hold the maxima of columns 8 j + 2 q4 + {0, 1}
    __syncwarp();
    if (lane < 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) mrow[8 * j + 2 * lane] = bm[2 * j], mrow[8 * j + 2 * lane + 1] = bm[2 * j + 1];
    }
    __syncwarp();
}

// The warp's MaxSim of finalist (off, len) (0 tokens: -inf), valid on lane
// 0: the maxima over every tile, then the in-order fp32 sum over the query
// tokens.  mrow: 32 floats of this warp.
template <int NB>
__device__ __forceinline__ float finalist(const IndexView& ix, const float* __restrict__ S, uint32_t rows, uint64_t off,
                                          uint32_t len, const uint2* qf, const uint32_t* lut, float* mrow) {
    finalist_max<NB>(ix, S, off, len, 0, 16, qf, lut, mrow);
    float total = 0.0f;
    if ((threadIdx.x & 31) == 0)
        for (uint32_t i = 0; i < rows; ++i) total = __fadd_rn(total, mrow[i]);
    __syncwarp();
    return total;
}

}  // namespace s4mma
}  // namespace plaid
