// range_stage2.cu — latency path: candidate generation (pipeline.cpp:52-87)
// and the pruned stage-2 centroid interaction (pipeline.cpp:97-137) in ONE
// launch, one CTA per pid range [r W, (r + 1) W), W ~ N / 148 (a power of two
// in [1K, 256K] ids: 64K and 135 ranges at 8.8M passages, one wave on 148 SMs).
//
// It replaces three kernels of the PDL chain (bitmap compaction, the
// kept-list accumulation into per-candidate rows, the stage-2 keys) and the
// N-bit bitmap + N-sized slot map they shared through HBM.  A sorted posting
// list's postings in a range are one run, located by the index-side range
// table (IndexView::range_tab).  Per CTA, in shared memory:
//   * the probed lists' runs set member bits (the union C1 of the probed
//     postings, restricted to the range);
//   * compaction in id order gives each member its rank; one atomic reserves
//     the range's slots in the stage-2 key array (key order is irrelevant to
//     the select that follows, which ranks keys, not positions);
//   * the kept lists' runs (t_cs keep bits, pipeline.cpp:89-95; at most 64
//     kept lists) set one bit per (member, kept list) in a 64-bit mask per
//     member — the member's set of distinct kept codes, all the max needs —
//     and a thread per member forms the key: per query token the max of
//     its kept lists' S rows (held in shared memory), then the in-order fp32
//     sum (0 without a kept token) — the same keys as the reference, bit
//     for bit (a warp-per-member grouping was latency-bound: ~14 us);
//   * the key histogram the stage-2 select starts from (SelectHist), and the
//     StageTrace counters (stage1_candidates, stage2_rows_gathered with the
//     postings' token multiplicities).
// Ranges whose runs overflow the shared-memory buffers, or queries keeping
// more than 64 centroids, score their members by scanning their codes
// (warp per member, masked), as the reference does.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr uint32_t kThreads = 1024;  // one CTA per SM: every warp hides the scoring's latency
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kKeptLists = 256;               // kept lists walked (more: code scan)
constexpr uint32_t kMaskWords = kKeptLists / 32;  // kept-list mask words per member
constexpr uint32_t kMaxLists = 256 + kKeptLists;
constexpr uint32_t kRangeWords = launch::kRangeIdsMax / 32;  // member bitmap words (widest range)
constexpr uint32_t kMCap = 2048;               // members per range (more: code scan)
constexpr uint32_t kPer = 4;                   // postings per thread per round
constexpr uint32_t kGCap = kPer * kThreads;    // kept postings per range (one register round)
constexpr uint32_t kMapCap = 8192;            // u16 flat -> list entries (longer ranges: binary search)

constexpr uint32_t kOffLCent = 0;
constexpr uint32_t kOffLStart = kOffLCent + kMaxLists * 4;
constexpr uint32_t kOffLPref = kOffLStart + kMaxLists * 8;
constexpr uint32_t kOffRBeg = kOffLPref + (kMaxLists + 4) * 4;
constexpr uint32_t kOffKS = kOffRBeg + kMaxLists * 4;
constexpr uint32_t kOffBm = kOffKS + kKeptLists * 33 * 4;
constexpr uint32_t kOffWpre = kOffBm + kRangeWords * 4;
constexpr uint32_t kOffMPid = kOffWpre + kRangeWords * 4;
constexpr uint32_t kOffMask = kOffMPid + kMCap * 4;                 // kMCap x kMaskWords u32: kept lists per member
constexpr uint32_t kOffMap = kOffMask + kMCap * kMaskWords * 4;      // kMapCap u16: flat posting -> list
constexpr uint32_t kOffUList = kOffMap + kMapCap * 2;                // kMCap u16: members with a kept token
constexpr uint32_t kSmemBytes = kOffUList + kMCap * 2;
static_assert(kRangeWords % kThreads == 0 && kMCap % kThreads == 0 && kThreads >= kMaxLists, "layout");
static_assert(kSmemBytes + sizeof(uint32_t) * 256 <= 227 * 1024, "shared memory budget");

struct Shared {
    uint32_t warp_tot[kWarps];
    uint32_t blk_s[32];
    uint32_t zeros, ucount, base, kept_n;
    uint32_t rows32;
    uint32_t kept_s[kKeptLists];
};

// Debug timeline (plaid_debug_rs2_trace): globaltimer at the phase
// boundaries of every CTA, when enabled.
__device__ int g_rs2_on;
__device__ unsigned long long g_rs2_t[512 * 8];
__device__ __forceinline__ void rs2_stamp(bool on, int k) {  // `on`: g_rs2_on, read once per CTA
    if (on && threadIdx.x == 0 && blockIdx.x < 512) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_rs2_t[blockIdx.x * 8 + k] = t;
    }
}

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < kWarps; ++w) {
        const uint32_t t = warp_tot[w];
        if (w < warp) before += t;
        tot += t;
    }
    __syncthreads();
    *total = tot;
    return before + incl - v;
}

// Key histogram of the stage-2 select (select_top_hist): bucket = top 16 key
// bits, warp-aggregated; the score-0 bucket and the per-2048-bucket block sums
// gathered in shared memory and flushed once per CTA.
__device__ __forceinline__ void hist_key(SelectHist* hs, uint64_t key, bool valid, Shared& sh) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t b = valid ? uint32_t(key >> kHistShift) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    if (valid && lane == uint32_t(__ffs(peers) - 1)) {
        if (b == kHistZeroBucket) atomicAdd(&sh.zeros, uint32_t(__popc(peers)));
        else {
            atomicAdd(&hs->hist[dev::hist_slot(b)], uint32_t(__popc(peers)));
            atomicAdd(&sh.blk_s[b >> 11], uint32_t(__popc(peers)));
        }
    }
}

// Masked scoring of one passage by a warp (pipeline.cpp:112-131 with the t_cs
// mask): score on every lane, *used = tokens on kept centroids.
__device__ __forceinline__ float score_masked(const uint32_t* __restrict__ codes, uint64_t off, uint32_t len,
                                             const float* __restrict__ S, uint32_t rows,
                                             const uint32_t* __restrict__ keep, uint32_t* used_out) {
    const uint32_t lane = threadIdx.x & 31;
    float acc = -INFINITY;
    uint32_t used = 0;
    for (uint32_t base = 0; base < len; base += 32) {
        const uint32_t t = base + lane;
        const uint32_t code = t < len ? __ldg(codes + off + t) : 0u;
        const bool valid = t < len && ((__ldg(keep + (code >> 5)) >> (code & 31)) & 1u);
        uint32_t bits = __ballot_sync(0xffffffffu, valid);
        used += __popc(bits);
        if (!bits) continue;
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
    if (used > 0)
        for (uint32_t j = 0; j < rows; ++j) total = __fadd_rn(total, __shfl_sync(0xffffffffu, acc, j));
    *used_out = used;
    return total;
}

__global__ void __launch_bounds__(kThreads, 1)
range_stage2_kernel(const IndexView ix, const float* __restrict__ S, uint32_t rows, const uint32_t* __restrict__ sel,
                    uint32_t nsel, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ kept,
                    const unsigned long long* __restrict__ kept_counts, uint64_t* __restrict__ keys_out,
                    unsigned long long* __restrict__ d_n1, unsigned long long* __restrict__ d_rows,
                    SelectHist* __restrict__ hs, uint64_t* __restrict__ ukeys, unsigned long long* __restrict__ d_nu) {
    const bool trace_on = g_rs2_on != 0;  // one load, in flight with the PDL wait
    rs2_stamp(trace_on, 6);  // CTA start (before the PDL wait)
    dev::pdl_wait();
    rs2_stamp(trace_on, 0);
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ Shared sh;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t r = blockIdx.x, R = ix.range_n, W = ix.range_w, WW = W / 32;
    const uint32_t base_pid = r * W;
    uint32_t* lcent = reinterpret_cast<uint32_t*>(smem + kOffLCent);
    uint64_t* lstart = reinterpret_cast<uint64_t*>(smem + kOffLStart);
    uint32_t* lpref = reinterpret_cast<uint32_t*>(smem + kOffLPref);
    uint32_t* rbeg = reinterpret_cast<uint32_t*>(smem + kOffRBeg);
    uint32_t* ks = reinterpret_cast<uint32_t*>(smem + kOffKS);
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem + kOffBm);
    uint32_t* wpre = reinterpret_cast<uint32_t*>(smem + kOffWpre);
    uint32_t* mpid = reinterpret_cast<uint32_t*>(smem + kOffMPid);
    uint32_t* mmask = reinterpret_cast<uint32_t*>(smem + kOffMask);
    uint16_t* map = reinterpret_cast<uint16_t*>(smem + kOffMap);
    uint16_t* ulist = reinterpret_cast<uint16_t*>(smem + kOffUList);
    uint32_t* kept_s = sh.kept_s;

    // the probed centroids (topn_postings: merge of the S_cq CTAs' top-nprobe
    // lists) and the kept list (its extra CTAs: the t_cs keep bits).  Folding
    // that merge into every CTA here was measured: +15 us, slower than the
    // separate launch's boundary
    const uint32_t kept_n = uint32_t(kept_counts[0]);
    const bool lists = kept_n <= kKeptLists;  // else every range scans its members' codes
    const uint32_t nk = lists ? kept_n : 0u;
    const uint32_t nl = nsel + nk;
    if (tid < nk) kept_s[tid] = __ldg(kept + tid);
    // (1) this range's run of every list, the kept centroids' S rows
    uint32_t cnt = 0;
    if (tid < nl) {
        const uint32_t c = tid < nsel ? __ldg(sel + tid) : __ldg(kept + (tid - nsel));
        lcent[tid] = c;
        lstart[tid] = __ldg(ix.ivf_offsets + c);
        const uint32_t* row = ix.range_tab + uint64_t(c) * (R + 1) + r;
        const uint32_t b = __ldg(row), e = __ldg(row + 1);
        rbeg[tid] = b;
        cnt = e - b;
    }
    __syncthreads();
    for (uint32_t j = warp; j < nk; j += kWarps)
        ks[j * 33 + lane] = dev::ord_f32(__ldg(S + uint64_t(kept_s[j]) * kScoresPitch + lane));
    for (uint32_t w = tid; w < WW; w += kThreads) bm[w] = 0u;
    // mask words in use: one per 32 kept lists, laid out [word][member]
    const uint32_t nwk = (nk + 31) / 32;
    for (uint32_t m = tid; m < nwk * kMCap; m += kThreads) mmask[m] = 0u;
    if (tid < 32) sh.blk_s[tid] = 0;
    if (tid == 0) sh.zeros = 0, sh.ucount = 0, sh.rows32 = 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(cnt, sh.warp_tot, &tot);
    if (tid < nl) lpref[tid] = ex;
    if (tid == 0) lpref[nl] = tot;
    const bool use_map = tot <= kMapCap;
    if (use_map && tid < nl)
        for (uint32_t i = 0; i < cnt; ++i) map[ex + i] = uint16_t(tid);
    __syncthreads();
    rs2_stamp(trace_on, 1);
    const uint32_t total_p = lpref[nsel], total = lpref[nl];
    auto locate = [&](uint32_t f, uint32_t lo, uint32_t hi) -> uint64_t {  // (list << 40) | posting index
        if (use_map) {
            lo = map[f];
        } else {
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (lpref[mid] <= f) lo = mid; else hi = mid;
            }
        }
        return (uint64_t(lo) << 40) | (lstart[lo] + rbeg[lo] + (f - lpref[lo]));
    };
    // (2) probed postings -> member bits; the kept postings' first round into
    // registers in the same pass (with their token multiplicities)
    const bool walk = lists && total - total_p <= kGCap;
    uint32_t kp[kPer], kl[kPer], km[kPer];
    for (uint32_t f0 = 0; f0 < total_p || (f0 == 0 && walk && total > total_p); f0 += kPer * kThreads) {
        uint32_t pp[kPer];
#pragma unroll
        for (int x = 0; x < int(kPer); ++x) {
            const uint32_t f = f0 + x * kThreads + tid;
            const uint64_t a1 = locate(f < total_p ? f : (total_p ? total_p - 1 : 0), 0, nsel);
            pp[x] = total_p ? __ldg(ix.ivf_postings + (a1 & 0xFFFFFFFFFFull)) : 0u;
            if (f0 == 0 && walk) {
                const uint32_t g = total_p + f;
                const bool in = g < total;
                const uint64_t a2 = locate(in ? g : (total > total_p ? total - 1 : 0), nsel, nl > nsel ? nl : nsel + 1);
                const uint64_t j = a2 & 0xFFFFFFFFFFull;
                kp[x] = in ? __ldg(ix.ivf_postings + j) : 0u;
                km[x] = in ? __ldg(ix.ivf_mult + j) : 0u;
                kl[x] = uint32_t(a2 >> 40) - nsel;
            }
        }
#pragma unroll
        for (int x = 0; x < int(kPer); ++x)
            if (f0 + x * kThreads + tid < total_p) {
                const uint32_t o = pp[x] - base_pid;
                atomicOr(bm + (o >> 5), 1u << (o & 31));
            }
    }
    __syncthreads();
    rs2_stamp(trace_on, 2);
    // (3) compaction: member ranks in id order; the range's key slots
    uint32_t m_r;
    {
        constexpr uint32_t kPW = kRangeWords / kThreads;  // words per thread at the widest range
        uint32_t v[kPW], mine = 0;
        const uint32_t w0 = tid * kPW;  // (narrower ranges: the high threads hold nothing)
#pragma unroll
        for (uint32_t j = 0; j < kPW; ++j) {
            v[j] = w0 + j < WW ? bm[w0 + j] : 0u;
            mine += __popc(v[j]);
        }
        uint32_t pos = block_excl_scan(mine, sh.warp_tot, &m_r);
#pragma unroll
        for (uint32_t j = 0; j < kPW; ++j) {
            if (w0 + j < WW) wpre[w0 + j] = pos;
            uint32_t x = v[j];
            while (x) {
                if (pos < kMCap) mpid[pos] = (w0 + j) * 32 + (__ffs(x) - 1);
                ++pos;
                x &= x - 1;
            }
        }
        if (tid == 0) sh.base = m_r ? uint32_t(atomicAdd(d_n1, (unsigned long long)m_r)) : 0u;
    }
    __syncthreads();
    rs2_stamp(trace_on, 3);
    const uint32_t kbase = sh.base;
    uint64_t* keys = keys_out + kbase;
    if (walk && m_r <= kMCap) {
        // (4) kept postings -> a 64-bit mask per member over the kept lists
        // (<= 64): the member's set of distinct kept codes is all the max
        // needs (pipeline.cpp:112-131)
        unsigned long long rows_local = 0;
#pragma unroll
        for (int x = 0; x < int(kPer); ++x) {
            if (total_p + x * kThreads + tid < total) {
                const uint32_t o = kp[x] - base_pid;
                const uint32_t wv = bm[o >> 5];
                if ((wv >> (o & 31)) & 1u) {
                    const uint32_t rk = wpre[o >> 5] + __popc(wv & ((1u << (o & 31)) - 1u));
                    atomicOr(mmask + (kl[x] >> 5) * kMCap + rk, 1u << (kl[x] & 31));
                    uint32_t m = km[x];
                    if (m == 255) {  // saturated multiplicity: recount from the codes
                        const uint32_t p = kp[x], c = lcent[nsel + kl[x]];
                        const uint64_t off = __ldg(ix.offsets + p);
                        const uint32_t len = __ldg(ix.doclens + p);
                        m = 0;
                        for (uint32_t t = 0; t < len; ++t) m += __ldg(ix.codes + off + t) == c;
                    }
                    rows_local += m;
                }
            }
        }
        // warp-reduced first: a 64-bit shared-memory atomic is a CAS loop
        uint32_t rl = uint32_t(rows_local);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rl += __shfl_xor_sync(0xffffffffu, rl, o);
        if (lane == 0 && rl) atomicAdd(&sh.rows32, rl);
        __syncthreads();
        rs2_stamp(trace_on, 4);
        // (5) members without a kept token: key 0; the others listed
        for (uint32_t m0 = 0; m0 < m_r; m0 += kThreads) {
            const uint32_t m = m0 + tid;
            bool z = false;
            uint64_t key = 0;
            if (m < m_r) {
                uint32_t any = 0;
#pragma unroll
                for (uint32_t q = 0; q < nwk; ++q) any |= mmask[q * kMCap + m];
                if (!any) {
                    z = true;
                    key = dev::make_key(0.0f, base_pid + mpid[m]);
                    keys[m] = key;
                }
            }
            // the members with a kept token, listed (one shared atomic per warp)
            const bool u = m < m_r && !z;
            const uint32_t ub = __ballot_sync(0xffffffffu, u);
            uint32_t b0 = 0;
            if (lane == 0 && ub) b0 = atomicAdd(&sh.ucount, __popc(ub));
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            if (u) ulist[b0 + __popc(ub & ((1u << lane) - 1u))] = uint16_t(m);
            hist_key(hs, key, z, sh);
        }
        __syncthreads();
        rs2_stamp(trace_on, 7);
        // (6) lane = listed member: the max over its kept lists' S rows (mask
        // bits; two halves of 16 query tokens in registers) and the in-order
        // sum (pipeline.cpp:125-131), all in the lane; the 32 members' row
        // loads proceed side by side.  (Lane = query token with a warp's
        // members one after another chained dependent loads per member.)
        const uint32_t nu = sh.ucount;
        // the range's slots in the list of keys with a kept token (read by the
        // stage-2 select when its boundary lies above score 0): one atomic per
        // CTA — one per warp put thousands of atomics on one L2 address
        if (tid == 0) sh.base = ukeys && nu ? uint32_t(atomicAdd(d_nu, (unsigned long long)nu)) : 0u;
        __syncthreads();
        const uint32_t ucta = sh.base;
        for (uint32_t u0 = warp * 32; u0 < nu; u0 += kWarps * 32) {
            const bool live = u0 + lane < nu;
            const uint32_t m = live ? ulist[u0 + lane] : 0u;
            float t = 0.0f;
#pragma unroll
            for (uint32_t h = 0; h < 2; ++h) {
                uint32_t mx[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) mx[j] = 0;
                for (uint32_t q = 0; live && q < nwk; ++q) {
                    for (uint32_t x = mmask[q * kMCap + m]; x; x &= x - 1) {
                        const uint32_t* row = ks + (q * 32 + uint32_t(__ffs(x) - 1)) * 33 + 16 * h;
#pragma unroll
                        for (int j = 0; j < 16; ++j) mx[j] = max(mx[j], row[j]);
                    }
                }
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (16 * h + j < rows) t = __fadd_rn(t, dev::unord_f32(mx[j]));
            }
            uint64_t key = 0;
            if (live) {
                const uint32_t pid = base_pid + mpid[m];
                key = dev::make_key(t, pid);
                keys[m] = key;
                if (ukeys) ukeys[ucta + u0 + lane] = key;
            }
            hist_key(hs, key, live, sh);
        }
    } else {        // code scan: a warp per member (bitmap order), masked interaction
        unsigned long long rows_local = 0;
        for (uint32_t w = warp; w < WW; w += kWarps) {
            uint32_t x = bm[w];
            while (x) {
                const uint32_t b = __ffs(x) - 1;
                x &= x - 1;
                const uint32_t pid = base_pid + w * 32 + b;
                uint32_t used;
                const float t = score_masked(ix.codes, __ldg(ix.offsets + pid), __ldg(ix.doclens + pid), S, rows,
                                             keep, &used);
                const uint64_t key = dev::make_key(t, pid);
                if (lane == 0) {
                    keys[wpre[w] + __popc(bm[w] & ((1u << b) - 1u))] = key;
                    if (ukeys) ukeys[atomicAdd(d_nu, 1ull)] = key;  // a superset of the positive keys
                }
                hist_key(hs, key, lane == 0, sh);
                rows_local += used;
            }
        }
        if (lane == 0 && rows_local) atomicAdd(&sh.rows32, uint32_t(rows_local));
    }
    __syncthreads();
    rs2_stamp(trace_on, 5);
    if (tid == 0) {
        if (sh.zeros) {
            atomicAdd(&hs->hist[dev::hist_slot(kHistZeroBucket)], sh.zeros);
            atomicAdd(&hs->blk[kHistZeroBucket >> 11], sh.zeros);
        }
        if (sh.rows32) atomicAdd(d_rows, (unsigned long long)sh.rows32);
    }
    if (tid < 32 && sh.blk_s[tid]) atomicAdd(&hs->blk[tid], sh.blk_s[tid]);
}

}  // namespace

namespace launch {

bool range_stage2_ok(const IndexView& ix, uint32_t rows, uint64_t nsel) {
    return ix.range_tab && rows <= 32 && nsel <= 256 && ix.N <= 0xFFFFFFFFull;
}

void range_stage2(const IndexView& ix, const float* d_scores, uint32_t rows, const uint32_t* d_sel, uint32_t nsel,
                  const uint32_t* d_keep_bits, const uint32_t* d_kept, const unsigned long long* d_kept_counts,
                  uint64_t* d_keys, uint64_t* d_n1, unsigned long long* d_rows, SelectHist* d_hist,
                  uint64_t* d_ukeys, uint64_t* d_nu, cudaStream_t st) {
    static PerDeviceOnce configured;
    if (configured.first())
        cudaFuncSetAttribute(range_stage2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    ::plaid::launch::pdl(range_stage2_kernel, ix.range_n, kThreads, kSmemBytes, st, ix, d_scores, rows, d_sel, nsel,
                         d_keep_bits, d_kept, d_kept_counts, d_keys, reinterpret_cast<unsigned long long*>(d_n1),
                         d_rows, d_hist, d_ukeys, reinterpret_cast<unsigned long long*>(d_nu));
    count_launch();
}

}  // namespace launch
}  // namespace plaid

// Debug: enable (out == NULL) or read back the range_stage2 timeline
// (out[512][8]: per CTA 0 start after the PDL wait, 1 runs located,
// 2 postings in, 3 compacted, 4 kept grouped, 5 scored, 6 launch-resident).
extern "C" int plaid_debug_rs2_trace(int enable, unsigned long long* out) {
    if (!out) return int(cudaMemcpyToSymbol(plaid::g_rs2_on, &enable, sizeof(int)));
    return int(cudaMemcpyFromSymbol(out, plaid::g_rs2_t, sizeof(plaid::g_rs2_t)));
}
