// device.cuh — device-side helpers shared by the PLAID kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace plaid {
namespace dev {

constexpr int kWarp = 32;
constexpr int kMaxRows = 32;  // |Q| <= 32: one query token per lane

// Orderable 32-bit image of an fp32 score: a > b (as floats) <=> ord(a) > ord(b).
// -0.0 is canonicalised to +0.0 first because the reference compares scores
// with `!=` / `>` (pipeline.cpp:147-150), for which the two zeros are equal.
__host__ __device__ __forceinline__ uint32_t ord_f32(float f) {
#ifdef __CUDA_ARCH__
    uint32_t u = __float_as_uint(f);
#else
    uint32_t u;
    __builtin_memcpy(&u, &f, 4);
#endif
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__host__ __device__ __forceinline__ float unord_f32(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    __builtin_memcpy(&f, &u, 4);
    return f;
#endif
}

// 64-bit selection key: larger key = better under (score desc, id asc), the
// total order of select_top (pipeline.cpp:147-150) and of the per-token
// centroid ranking (pipeline.cpp:67-72).  Keys are unique for unique ids.
__host__ __device__ __forceinline__ uint64_t make_key(float score, uint32_t id) {
    return (uint64_t(ord_f32(score)) << 32) | uint64_t(~id);
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t key) { return ~uint32_t(key); }
__host__ __device__ __forceinline__ float key_score(uint64_t key) { return unord_f32(uint32_t(key >> 32)); }

// In-order fp32 multiply-then-add, never contracted into an FMA: the
// reference's `acc += a[i] * b[i]` (types.hpp:18-22).
__device__ __forceinline__ float madd_rn(float acc, float a, float b) {
    return __fadd_rn(acc, __fmul_rn(a, b));
}

// (a.x * s, a.y * s), each rounded to nearest: one FMUL2 on sm_100.  Only
// the multiply is packed — ptxas contracts a packed mul.rn.f32x2 feeding a
// packed add.rn.f32x2 into FFMA2 (checked with cuobjdump), which would break
// the reference's separately rounded multiply-then-add, so the adds stay
// scalar __fadd_rn.
__device__ __forceinline__ float2 mul2_rn(float2 a, float s) {
    unsigned long long r;
    const float2 b = make_float2(s, s);
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
          "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&r);
}

// `if (s > acc) acc = s` (pipeline.cpp:122, maxsim.cpp:95).
__device__ __forceinline__ float max_gt(float acc, float s) { return s > acc ? s : acc; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max_gt(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: every kernel is launched with
// programmatic stream serialization (launch::pdl) so its launch and block
// scheduling overlap the previous kernel's tail; it must not touch memory the
// previous kernels write before this wait (a no-op without a PDL edge).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// "Last CTA out" ticket: one thread per CTA, after a __syncthreads that
// follows the CTA's global reads and writes.  acq_rel at gpu scope: releases
// this CTA's accesses (ordered before it by the barrier) and acquires every
// earlier ticket holder's, without the sequentially consistent fence
// (MEMBAR.SC + L1 invalidate) that __threadfence() costs.  True for the last
// of `n` CTAs.
__device__ __forceinline__ bool last_ticket(unsigned int* ticket, unsigned int n) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
    return old == n - 1;
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// *dst += the sum over the block's warps of lane 0's v: one global atomic per
// CTA instead of one per warp (thousands of same-address atomics queue on one
// L2 slice).  Every thread of the block must call it.
__device__ __forceinline__ void block_add_lane0(unsigned long long* dst, unsigned long long v) {
    __shared__ unsigned long long tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    if ((threadIdx.x & 31u) == 0 && v) atomicAdd(&tot, v);
    __syncthreads();
    if (threadIdx.x == 0 && tot) atomicAdd(dst, tot);
}

// Slot of key bucket b in SelectHist::hist: each 2048-bucket block is stored
// transposed (bucket 32 j + l at 64 l + j), so the run of consecutive buckets
// a query's scores fill is spread over 32 cache lines instead of a few — the
// producers' histogram atomics otherwise queue on one L2 slice.  Block sums
// are unchanged; hist_find walks a block through shared memory.
__device__ __forceinline__ uint32_t hist_slot(uint32_t b) {
    return (b & ~0x7FFu) | ((b & 31u) << 6) | ((b >> 5) & 63u);
}

// Branchless insertion of x into a descending list k[0..NP) of unique keys.
template <int NP>
__device__ __forceinline__ void topn_insert(uint64_t (&k)[NP], uint64_t x) {
    if (x <= k[NP - 1]) return;
#pragma unroll
    for (int j = NP - 1; j > 0; --j) {
        uint64_t lo = x < k[j - 1] ? x : k[j - 1];
        k[j] = k[j] > lo ? k[j] : lo;
    }
    k[0] = k[0] > x ? k[0] : x;
}

}  // namespace dev
}  // namespace plaid
