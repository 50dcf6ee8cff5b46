// select.cu — select_top (pipeline.cpp:139-163) on 64-bit keys.
//
// Keys pack (ord(score) << 32 | ~id), so "largest key first" is exactly the
// reference's (score desc, id asc) order and every key is unique.  Two paths:
//   * select_top_large: multi-CTA radix select (6 digit passes of <= 11 bits
//     over the 64-bit key; the last CTA of each pass picks the digit, so there
//     is no host round trip) followed by a compaction of the keys >= the
//     threshold.  Used for stage 2 where the input is the whole candidate set.
//   * sort_top: one CTA bitonic sort in shared memory (<= 8192 keys), or a
//     global-memory bitonic network beyond that; emits the first `want` keys
//     as (id, score) pairs in order.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr uint32_t kBins = 2048;
constexpr int kPasses = 6;
__host__ __device__ constexpr int pass_shift(int p) { return p < 5 ? 53 - 11 * p : 0; }
__host__ __device__ constexpr int pass_bits(int p) { return p < 5 ? 11 : 9; }

__global__ void sel_init_kernel(SelectState* st, const uint64_t* __restrict__ d_n, uint64_t want,
                                uint64_t* __restrict__ out_n) {
    const uint64_t n = *d_n;
    for (uint32_t b = threadIdx.x; b < kBins; b += blockDim.x) st->hist[b] = 0;
    if (threadIdx.x == 0) {
        st->prefix = 0;
        st->mask = 0;
        st->remaining = n < want ? n : want;
        st->done = n <= want ? 1u : 0u;
        st->ticket = 0;
        *out_n = 0;
    }
}

__global__ void __launch_bounds__(256)
sel_pass_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                SelectState* st, int pass) {
    __shared__ uint32_t h[kBins];
    __shared__ uint32_t part[256];
    __shared__ bool last;
    if (*((volatile unsigned int*)&st->done)) return;
    const int shift = pass_shift(pass);
    const uint32_t nb = 1u << pass_bits(pass);
    const uint64_t prefix = st->prefix, mask = st->mask;
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const uint64_t n = *d_n;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[i];
        if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & (nb - 1)], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
        if (h[b]) atomicAdd(&st->hist[b], h[b]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // Last CTA: find the digit holding the remaining-th largest key.
    const uint32_t per = nb / blockDim.x;  // bins per thread (8 or 2)
    // thread t owns bins [nb - (t+1)*per, nb - t*per) (descending order)
    uint32_t s = 0;
    for (uint32_t j = 0; j < per; ++j) s += __ldcg(&st->hist[nb - 1 - (threadIdx.x * per + j)]);
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t rem = st->remaining;
        uint64_t cum = 0;
        uint32_t t = 0;
        for (; t < blockDim.x; ++t) {
            if (cum + part[t] >= rem) break;
            cum += part[t];
        }
        uint32_t bin = 0;
        uint32_t cnt = 0;
        for (uint32_t j = 0; j < per; ++j) {
            bin = nb - 1 - (t * per + j);
            cnt = __ldcg(&st->hist[bin]);
            if (cum + cnt >= rem) break;
            cum += cnt;
        }
        const uint64_t left = rem - cum;
        st->remaining = left;
        st->prefix = prefix | (uint64_t(bin) << shift);
        st->mask = mask | (uint64_t(nb - 1) << shift);
        if (cnt == left) st->done = 1u;
        st->ticket = 0;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < kBins; b += blockDim.x) st->hist[b] = 0;
}

__global__ void __launch_bounds__(256)
sel_compact_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                   const SelectState* st, uint64_t* __restrict__ out, uint64_t* __restrict__ out_n) {
    const uint64_t thr = st->prefix;
    const uint64_t n = *d_n;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t i0 = blockIdx.x * uint64_t(blockDim.x); i0 < n; i0 += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = i0 + threadIdx.x;
        const uint64_t k = i < n ? keys[i] : 0;
        const bool take = i < n && k >= thr;
        const uint32_t ballot = __ballot_sync(0xffffffffu, take);
        if (!ballot) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd((unsigned long long*)out_n, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) out[base + __popc(ballot & ((1u << lane) - 1))] = k;
    }
}

// Emit the first min(want, n) keys of a descending array.
__device__ __forceinline__ void emit(uint64_t j, uint64_t key, uint64_t* out_keys, uint32_t* out_ids,
                                     float* out_scores, uint32_t id_base) {
    if (out_keys) out_keys[j] = key;
    if (out_ids) out_ids[j] = dev::key_id(key) + id_base;
    if (out_scores) out_scores[j] = dev::key_score(key);
}

__global__ void __launch_bounds__(1024)
sort_small_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n, uint32_t npad,
                  uint64_t want, uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_ids,
                  float* __restrict__ out_scores, uint64_t* __restrict__ out_n, uint32_t id_base) {
    extern __shared__ uint64_t s[];
    const uint64_t n = *d_n;
    for (uint32_t i = threadIdx.x; i < npad; i += blockDim.x) s[i] = i < n ? keys[i] : 0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= npad; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < npad; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = s[i], b = s[ixj];
                    const bool desc = (i & k) == 0;
                    if (desc ? (a < b) : (a > b)) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    const uint64_t m = n < want ? n : want;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) emit(j, s[j], out_keys, out_ids, out_scores, id_base);
    if (threadIdx.x == 0 && out_n) *out_n = m;
}

__global__ void pad_copy_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ d_n,
                                uint64_t npad, uint64_t* __restrict__ tmp) {
    const uint64_t n = *d_n;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < npad;
         i += uint64_t(gridDim.x) * blockDim.x)
        tmp[i] = i < n ? keys[i] : 0ull;
}

__global__ void bitonic_step_kernel(uint64_t* __restrict__ s, uint64_t npad, uint64_t j, uint64_t k) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < npad;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t ixj = i ^ j;
        if (ixj > i) {
            const uint64_t a = s[i], b = s[ixj];
            const bool desc = (i & k) == 0;
            if (desc ? (a < b) : (a > b)) {
                s[i] = b;
                s[ixj] = a;
            }
        }
    }
}

__global__ void emit_kernel(const uint64_t* __restrict__ sorted, const uint64_t* __restrict__ d_n,
                            uint64_t want, uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_ids,
                            float* __restrict__ out_scores, uint64_t* __restrict__ out_n, uint32_t id_base) {
    const uint64_t n = *d_n;
    const uint64_t m = n < want ? n : want;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < m;
         j += uint64_t(gridDim.x) * blockDim.x)
        emit(j, sorted[j], out_keys, out_ids, out_scores, id_base);
    if (blockIdx.x == 0 && threadIdx.x == 0 && out_n) *out_n = m;
}

__global__ void make_keys_kernel(const uint32_t* __restrict__ ids, const float* __restrict__ scores,
                                 uint64_t n, uint64_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        keys[i] = dev::make_key(scores[i], ids[i]);
}

// Per shard g, entries [0, counts[g]) of row g (stride) become keys; the rest
// of the G*stride slots are 0 (below every real key).
__global__ void merge_keys_kernel(const uint32_t* __restrict__ pids, const float* __restrict__ scores,
                                  const uint64_t* __restrict__ counts, uint64_t shards, uint64_t stride,
                                  uint64_t* __restrict__ keys, uint64_t* __restrict__ d_n) {
    const uint64_t total = shards * stride;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = i / stride, j = i % stride;
        keys[i] = j < counts[g] ? dev::make_key(scores[i], pids[i]) : 0ull;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *d_n = total;
}

__global__ void copy_count_kernel(const uint64_t* src, uint64_t* dst, uint64_t cap) {
    const uint64_t v = *src;
    *dst = v < cap ? v : cap;
}

__global__ void validate_query_kernel(const float* __restrict__ q, uint32_t rows, uint32_t dim,
                                      int* __restrict__ status) {
    const uint32_t r = threadIdx.x;
    if (r >= rows) return;
    double acc = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
        const double v = double(q[r * dim + d]);
        acc = __dadd_rn(acc, __dmul_rn(v, v));
    }
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

}  // namespace

namespace launch {

void select_top_large(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want,
                      SelectState* d_state, uint64_t* d_out_keys, uint64_t* d_out_n,
                      cudaStream_t st) {
    sel_init_kernel<<<1, 256, 0, st>>>(d_state, d_n, want, d_out_n);
    count_launch();
    const uint32_t grid = grid_for(nmax, 256, uint32_t(sm_count()) * 4);
    for (int p = 0; p < kPasses; ++p) {
        sel_pass_kernel<<<grid, 256, 0, st>>>(d_keys, d_n, d_state, p);
        count_launch();
    }
    sel_compact_kernel<<<grid, 256, 0, st>>>(d_keys, d_n, d_state, d_out_keys, d_out_n);
    count_launch();
}

uint64_t sort_tmp_capacity(uint64_t nmax) { return nmax <= kSmallSortMax ? 0 : next_pow2(nmax); }

void sort_top(const uint64_t* d_keys, const uint64_t* d_n, uint64_t nmax, uint64_t want,
              uint64_t* d_out_keys, uint32_t* d_out_ids, float* d_out_scores, uint64_t* d_out_n,
              uint32_t id_base, uint64_t* d_tmp, cudaStream_t st) {
    if (nmax <= kSmallSortMax) {
        const uint32_t npad = uint32_t(next_pow2(nmax < 2 ? 2 : nmax));
        const size_t smem = size_t(npad) * sizeof(uint64_t);
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(sort_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kSmallSortMax * sizeof(uint64_t)));
            configured = true;
        }
        sort_small_kernel<<<1, 1024, smem, st>>>(d_keys, d_n, npad, want, d_out_keys, d_out_ids,
                                                 d_out_scores, d_out_n, id_base);
        count_launch();
        return;
    }
    const uint64_t npad = next_pow2(nmax);
    const uint32_t grid = grid_for(npad, 256, uint32_t(sm_count()) * 8);
    pad_copy_kernel<<<grid, 256, 0, st>>>(d_keys, d_n, npad, d_tmp);
    count_launch();
    for (uint64_t k = 2; k <= npad; k <<= 1)
        for (uint64_t j = k >> 1; j > 0; j >>= 1) {
            bitonic_step_kernel<<<grid, 256, 0, st>>>(d_tmp, npad, j, k);
            count_launch();
        }
    emit_kernel<<<grid_for(want, 256, 4096), 256, 0, st>>>(d_tmp, d_n, want, d_out_keys, d_out_ids,
                                                          d_out_scores, d_out_n, id_base);
    count_launch();
}

void make_keys(const uint32_t* d_ids, const float* d_scores, uint64_t n, uint64_t* d_keys,
               cudaStream_t st) {
    make_keys_kernel<<<grid_for(n, 256, 4096), 256, 0, st>>>(d_ids, d_scores, n, d_keys);
    count_launch();
}

void merge_topk(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts,
                uint64_t shards, uint64_t stride, uint64_t k, uint64_t* d_tmp_keys, uint64_t* d_tmp_n,
                uint32_t* d_out_pids, float* d_out_scores, uint64_t* d_out_n, uint64_t* d_sort_tmp,
                cudaStream_t st) {
    merge_keys_kernel<<<grid_for(shards * stride, 256, 4096), 256, 0, st>>>(
        d_pids, d_scores, d_counts, shards, stride, d_tmp_keys, d_tmp_n);
    count_launch();
    sort_top(d_tmp_keys, d_tmp_n, shards * stride, k, nullptr, d_out_pids, d_out_scores, d_out_n, 0,
             d_sort_tmp, st);
}

void copy_count(const uint64_t* src, uint64_t* dst, uint64_t cap, cudaStream_t st) {
    copy_count_kernel<<<1, 1, 0, st>>>(src, dst, cap);
    count_launch();
}

void validate_query(const float* d_q, uint32_t rows, uint32_t dim, int* d_status, cudaStream_t st) {
    validate_query_kernel<<<1, 32, 0, st>>>(d_q, rows, dim, d_status);
    count_launch();
}

}  // namespace launch
}  // namespace plaid
