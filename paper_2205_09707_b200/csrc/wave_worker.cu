// wave_worker.cu — throughput-mode stages 1b-4: one CTA per query runs the
// rest of lir::search (pipeline.cpp:232-283) after the wave's S_cq pass
// (wave_scores.cu, or the exact per-query S_cq in EXACT mode).
//
// The latency path spreads ONE query over the whole GPU in a chain of ~14
// kernels; in throughput mode hundreds of queries are in flight, so each
// query gets one CTA and block-level primitives, the wave is one launch, and
// no query ever waits on a grid-wide step.  Everything after S is the
// reference's arithmetic, so given the same S the results are bit-identical
// to lir::search (tests/test_gpu_wave.py runs it on the exact S_cq).
//
// Per query (CTA, 256 threads):
//   A  top-nprobe per query token: merge of the S_cq pass's partial lists
//      (keys (score, ~id): the reference's (score desc, id asc) order,
//      pipeline.cpp:67-72); kept-centroid list from the keep bits.
//   B-E candidate generation and stage 2 over pid ranges of W = 64K ids.
//      Every posting list is sorted, so a list's postings in a range are one
//      run, located by the index-side range table (range_tab, built once per
//      index).  Per range, in shared memory: the probed postings set member
//      bits; the members are compacted in id order (= the reference's sort,
//      pipeline.cpp:83); the kept postings are grouped by member with a
//      counting sort; a member's stage-2 score is the in-order sum over the
//      query tokens of the max of its kept centroids' S rows (a max needs
//      only the member's set of distinct kept codes, and p owns code c iff p
//      is in postings(c)), 0 without one.  Nothing per query is N-sized and
//      no global atomics are needed, so hundreds of queries in flight do not
//      thrash L2.  Many or long kept lists (t_cs near -1) or overfull
//      ranges: a warp per candidate scans its codes instead
//      (pipeline.cpp:97-137 literally).
//      Top-ndocs SET by a CTA radix select (11-bit digits, shared-memory
//      histogram, boundary bucket carried to the next digit); when at least
//      ndocs rows have a positive score only those rows are candidates.
//   F  stage 3: warp per survivor stream (the warp's passages laid end to
//      end), 32 S-row gathers in flight, running max per query token reset
//      at passage starts; keys; the top-stage3_width SET.
//   G  stage 4 (residual_codec.cpp:97-132, maxsim.cpp:66-104): warp per
//      finalist, four tokens per step: v = C[code] + w[bucket] (4 dims per
//      lane), v *= inv (the reference's fp64 norm, precomputed per token at
//      index load), lane = query token: four in-order fp32 dot chains,
//      running max, in-order sum.  Exact arithmetic, bit-identical scores.
//   H  bitonic sort of the finalists' keys in shared memory, top-k out.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"
#include "s4_mma.cuh"

namespace plaid {
namespace {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kKeptCap = 256;           // kept centroids listed per query
constexpr uint32_t kKeptLists = 64;          // kept lists walked range by range (more: code scan)
constexpr uint64_t kListsPerCandidate = 4;   // kept postings per probed posting above which stage 2 scans codes
constexpr uint32_t kQPitch = 132;            // floats per query row in shared memory (16-B aligned, conflict-free)
constexpr uint32_t kSortCap = launch::kWaveSortCap;
constexpr uint32_t kRangeWords = launch::kWaveRangeIds / 32;  // member bitmap words per range
constexpr uint32_t kPer = 8;                 // postings per thread per round
constexpr uint32_t kMaxLists = 256 + kKeptLists;
constexpr uint32_t kMCap = 2048;             // C1 members per range (bounded by the range's probed postings)
constexpr uint32_t kGCap = kPer * kThreads;  // kept postings per range (one register chunk)

// shared-memory layout (bytes); phases A-E and F-H reuse the same space
constexpr uint32_t kOffProbe = 0;                                  // 256 u32
constexpr uint32_t kOffKept = kOffProbe + 256 * 4;                 // kKeptCap u32
constexpr uint32_t kOffLCent = kOffKept + kKeptCap * 4;            // kMaxLists u32: list centroids
constexpr uint32_t kOffLStart = kOffLCent + kMaxLists * 4;         // kMaxLists u64: list starts
constexpr uint32_t kOffLPref = kOffLStart + kMaxLists * 8;         // kMaxLists + 1 u32: run prefix over the lists
constexpr uint32_t kOffRBeg = kOffLPref + (kMaxLists + 4) * 4;     // kMaxLists u32: run start per list
constexpr uint32_t kOffKS = kOffRBeg + kMaxLists * 4;              // kKeptLists x 33 u32
constexpr uint32_t kOffBm = kOffKS + kKeptLists * 33 * 4;          // kRangeWords u32
constexpr uint32_t kOffWpre = kOffBm + kRangeWords * 4;            // kRangeWords u16
constexpr uint32_t kOffMPid = kOffWpre + kRangeWords * 2;          // kMCap u16
constexpr uint32_t kOffGOff = kOffMPid + kMCap * 2;                // kMCap + 1 u16
constexpr uint32_t kOffGrp = kOffGOff + (kMCap + 8) * 2;           // kGCap u16
constexpr uint32_t kOffUList = kOffGrp + kGCap * 2;                // kMCap u16: members with kept tokens
constexpr uint32_t kOffTile = kOffUList + kMCap * 2;               // kWarps x 16 x 33 u32
constexpr uint32_t kOffHist = kOffTile + kWarps * 16 * 33 * 4;    // 2048 u32 (A-F)
constexpr uint32_t kMapCap = kWarps * 16 * 33 * 2;                 // u16 flat->list map entries (tile space)
constexpr uint32_t kEndAE = kOffHist + 2048 * 4;
constexpr uint32_t kOffQ = 0;                                      // 32 x kQPitch f32 (G)
constexpr uint32_t kTok = 2;                                       // stage-4 tokens per warp step
constexpr uint32_t kOffV = kOffQ + 32 * kQPitch * 4;               // kWarps x kTok x 128 f32 (G)
constexpr uint32_t kOffK4 = kOffV + kWarps * kTok * 128 * 4;       // kSortCap u64 (G-H)
constexpr uint32_t kEndGH = kOffK4 + kSortCap * 8;
// G on the tensor cores (WaveArgs::s4_tensor): Q's bf16 hi/lo B fragments,
// the residual-pair LUTs and a per-warp row of maxima, past the exact G/H layout
constexpr uint32_t kOffQF = kEndGH;                                 // s4mma::kQFragBytes
constexpr uint32_t kOffLut = kOffQF + 8 * 4 * 2 * 32 * 8;           // s4mma::kLutBytes
constexpr uint32_t kOffMaxRow = kOffLut + 2 * 256 * 4;              // kWarps x 32 f32
constexpr uint32_t kEndG2 = kOffMaxRow + kWarps * 32 * 4;
constexpr uint32_t kSmemBytes = kEndAE > kEndGH ? (kEndAE > kEndG2 ? kEndAE : kEndG2) : (kEndGH > kEndG2 ? kEndGH : kEndG2);
static_assert(kRangeWords % kThreads == 0 && 2 * kThreads >= kMaxLists, "range words / lists per thread");

struct Shared {
    uint32_t kept_n, nsel, n1, tmp;
    unsigned long long kept_post, probed_post;
    uint32_t maxp, maxk, ucount;
    uint32_t bnd_bin, bnd_above, outn, sidn;
    uint32_t warp_tot[kWarps];
    uint32_t zero_cnt, nused, npos;
    int bad;
};

// Phase timeline (launch::WaveArgs::trace): globaltimer at the phase
// boundaries of each query's CTA, for tools/wave_probe.py.
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void stamp(const launch::WaveArgs& a, uint32_t qi, uint32_t k) {
    if (a.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[uint64_t(qi) * 16 + k] = t;
    }
}

// (a.x * b.x, a.y * b.y), each rounded to nearest: one FMUL2 (the adds stay
// separate, so nothing is contracted into an FMA)
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&r);
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
    __syncthreads();  // warp_tot reusable
    *total = tot;
    return before + incl - v;
}

// Top `want` of keys[0..n) (unique) into out[0..min(n, want)), unordered:
// MSB radix select, 11-bit digits (shifts 53, 42, 31, 20, 9, then 9 bits at
// 0), shared-memory histogram, keys of the boundary digit carried to the next
// level in a side buffer.  hist (2048 u32) holds the level-0 histogram when
// hist_ready, else it is built here.  Every thread must call it.
__device__ uint32_t cta_select(const uint64_t* keys, uint32_t n, uint32_t want, uint64_t* out, uint64_t* side0,
                               uint64_t* side1, uint32_t* hist, Shared& sh, bool hist_ready) {
    const uint32_t tid = threadIdx.x;
    if (n <= want) {
        for (uint32_t i = tid; i < n; i += kThreads) out[i] = __ldcg(keys + i);
        __syncthreads();
        return n;
    }
    if (tid == 0) sh.outn = 0;
    const uint64_t* cur = keys;
    uint32_t cn = n, rem = want;
    int shift = 53;
    int ping = 0;
    bool ready = hist_ready;
    while (true) {
        const uint32_t mask = shift == 0 ? 511u : 2047u;
        if (!ready) {
            for (uint32_t b = tid; b < 2048; b += kThreads) hist[b] = 0;
            __syncthreads();
            for (uint32_t i = tid; i < cn; i += kThreads) atomicAdd(&hist[(__ldcg(cur + i) >> shift) & mask], 1u);
        }
        ready = false;
        __syncthreads();
        // thread t owns bins 2047 - 8t .. 2040 - 8t (descending)
        uint32_t c[8], s = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = hist[2047 - 8 * tid - j], s += c[j];
        uint32_t tot;
        uint32_t run = block_excl_scan(s, sh.warp_tot, &tot);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (run < rem && run + c[j] >= rem) {
                sh.bnd_bin = 2047 - 8 * tid - j;
                sh.bnd_above = run;
            }
            run += c[j];
        }
        __syncthreads();
        const uint32_t b = sh.bnd_bin, above = sh.bnd_above, cb = hist[b];
        if (!(above == 0 && cb == cn)) {  // else every key shares this digit: nothing to move
            if (tid == 0) sh.sidn = 0;
            __syncthreads();
            uint64_t* dst = ping ? side1 : side0;
            for (uint32_t i = tid; i < cn; i += kThreads) {
                const uint64_t k = __ldcg(cur + i);
                const uint32_t d = uint32_t(k >> shift) & mask;
                if (d > b) out[atomicAdd(&sh.outn, 1u)] = k;
                else if (d == b) dst[atomicAdd(&sh.sidn, 1u)] = k;
            }
            __syncthreads();
            cur = dst;
            ping ^= 1;
            cn = cb;
        }
        rem -= above;
        if (rem == cn) {
            const uint32_t o = sh.outn;
            for (uint32_t i = tid; i < cn; i += kThreads) out[o + i] = __ldcg(cur + i);
            __syncthreads();
            return want;
        }
        shift = shift >= 11 ? shift - 11 : 0;
        __syncthreads();
    }
}

// Stage-3 scoring of one passage by a warp (pipeline.cpp:112-131, no mask):
// score on every lane, *used = tokens.
__device__ __forceinline__ float score_passage(const uint32_t* __restrict__ codes, uint64_t off, uint32_t len,
                                              const float* __restrict__ S, uint32_t rows,
                                              const uint32_t* __restrict__ keep, bool masked, uint32_t* used_out) {
    const uint32_t lane = threadIdx.x & 31;
    float acc = -INFINITY;
    uint32_t used = 0;
    for (uint32_t base = 0; base < len; base += 32) {
        const uint32_t t = base + lane;
        const uint32_t code = t < len ? __ldg(codes + off + t) : 0u;
        bool valid = t < len;
        if (masked) valid = valid && ((__ldg(keep + (code >> 5)) >> (code & 31)) & 1u);
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

// Stage 4 on the tensor cores (TENSOR score mode): s4_mma.cuh's warp scorer
// (r_t . q_i on mma.sync, (S + r.q) * inv, max over the tokens, in-order
// sum), a warp per finalist w, w + 8, ...; keys into k4.
template <int NB>
__device__ __forceinline__ void stage4_tensor(const IndexView& ix, const launch::WaveArgs& a, const float* __restrict__ Q,
                                           const float* __restrict__ S, uint32_t rows, uint32_t n3,
                                           const uint64_t* __restrict__ sel3, uint64_t* f_off, uint32_t* f_len,
                                           uint8_t* smem) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint2* qf = reinterpret_cast<uint2*>(smem + kOffQF);
    uint32_t* lut = reinterpret_cast<uint32_t*>(smem + kOffLut);
    float* mrow = reinterpret_cast<float*>(smem + kOffMaxRow) + warp * 32;
    uint64_t* k4 = reinterpret_cast<uint64_t*>(smem + kOffK4);
    s4mma::setup<NB>(ix, Q, rows, qf, lut);
    for (uint32_t i = tid; i < n3; i += kThreads) {
        const uint32_t pid = dev::key_id(__ldcg(sel3 + i));
        f_off[i] = __ldg(ix.offsets + pid);
        f_len[i] = __ldg(ix.doclens + pid);
    }
    __threadfence_block();
    __syncthreads();
    for (uint32_t f = warp; f < n3; f += kWarps) {
        const float total = s4mma::finalist<NB>(ix, S, rows, f_off[f], f_len[f], qf, lut, mrow);
        if (lane == 0) k4[f] = dev::make_key(total, dev::key_id(__ldcg(sel3 + f)));
    }
}

template <int NP, int NB>
__global__ void __launch_bounds__(kThreads, 3) wave_worker_kernel(const IndexView ix, const launch::WaveArgs a) {
    dev::pdl_wait();
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ Shared sh;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t qi = blockIdx.x;
    const uint32_t rows = a.rows;
    const float* __restrict__ Q = a.Q + uint64_t(qi) * rows * 128;
    const float* __restrict__ S = a.S + uint64_t(qi) * a.s_stride;
    const uint32_t* __restrict__ keep = a.keep + uint64_t(qi) * a.keep_stride;
    uint32_t* __restrict__ c1 = a.c1 + uint64_t(qi) * a.c1cap;
    uint32_t* __restrict__ acc = a.acc + uint64_t(qi) * a.ndocs * 32;  // stage-3 maxima rows (zero between queries)
    uint64_t* __restrict__ keys = a.keys + uint64_t(qi) * a.c1cap;
    uint64_t* __restrict__ side0 = a.side + uint64_t(qi) * a.c1cap * 3;
    uint64_t* __restrict__ side1 = side0 + a.c1cap;
    uint64_t* __restrict__ sel2 = a.sel + uint64_t(qi) * a.sel_stride;
    uint64_t* __restrict__ sel3 = sel2 + a.ndocs;
    uint32_t* probe = reinterpret_cast<uint32_t*>(smem + kOffProbe);
    uint32_t* kept = reinterpret_cast<uint32_t*>(smem + kOffKept);
    const uint64_t K = ix.K;

    if (tid == 0) {
        sh.kept_n = 0, sh.kept_post = 0, sh.probed_post = 0, sh.bad = 0;
    }
    stamp(a, qi, 0);
    // ---- 0: device-side query validation (types.cpp:61-72; in-order fp64)
    if (a.validate && warp == 0 && lane < rows) {
        double s = 0.0;
        for (uint32_t d = 0; d < 128; ++d) {
            const double v = double(__ldg(Q + lane * 128 + d));
            s = __dadd_rn(s, __dmul_rn(v, v));
        }
        if (fabs(sqrt(s) - 1.0) > double(1e-3f)) sh.bad = 1;
    }
    __syncthreads();
    if (sh.bad) {
        if (tid == 0) {
            atomicExch(a.status, 2);  // NotNormalized + 1
            a.out_n[qi] = 0;
        }
        return;
    }

    // ---- A: top-nprobe per query token; kept-centroid list
    for (uint32_t i = warp; i < rows; i += kWarps) {
        uint64_t top[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) top[j] = 0;
        const uint64_t* P = a.partial + uint64_t(qi) * a.partial_stride;
        for (uint32_t l = lane; l < a.nlists; l += 32) {
            uint64_t v[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) v[j] = __ldcg(P + (uint64_t(l) * 32 + i) * NP + j);
#pragma unroll
            for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, v[j]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t pv[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) pv[j] = __shfl_xor_sync(0xffffffffu, top[j], o);
#pragma unroll
            for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, pv[j]);
        }
        unsigned long long len = 0;
#pragma unroll
        for (int j = 0; j < NP; ++j)
            if (uint32_t(j) < a.nprobe) {
                const uint32_t c = dev::key_id(top[j]);
                if (lane == 0) probe[i * a.nprobe + j] = c;
                len += __ldg(ix.ivf_offsets + c + 1) - __ldg(ix.ivf_offsets + c);
            }
        if (lane == 0) atomicAdd(&sh.probed_post, len);
    }
    {
        const uint32_t nkw = uint32_t((K + 31) / 32);
        unsigned long long my_post = 0;
        for (uint32_t w0 = 0; w0 < nkw; w0 += 8 * kThreads) {
            uint32_t kwv[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                const uint32_t w = w0 + x * kThreads + tid;
                kwv[x] = w < nkw ? __ldcg(keep + w) : 0u;
            }
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                uint32_t kw = kwv[x];
                while (kw) {
                    const uint32_t c = (w0 + x * kThreads + tid) * 32 + (__ffs(kw) - 1);
                    kw &= kw - 1;
                    const uint32_t slot = atomicAdd(&sh.kept_n, 1u);
                    if (slot < kKeptCap) kept[slot] = c;
                    my_post += __ldg(ix.ivf_offsets + c + 1) - __ldg(ix.ivf_offsets + c);
                }
            }
        }
        if (my_post) atomicAdd(&sh.kept_post, my_post);
    }
    __syncthreads();
    const uint32_t nprobed = rows * a.nprobe;
    const uint32_t kept_n = sh.kept_n;
    // stage 2 walks the kept lists range by range unless they are many or
    // long (t_cs near -1): then a warp per candidate scans its codes
    uint32_t* lcent = reinterpret_cast<uint32_t*>(smem + kOffLCent);  // list centroid: probed, then kept
    uint64_t* lstart = reinterpret_cast<uint64_t*>(smem + kOffLStart);
    uint32_t* lpref = reinterpret_cast<uint32_t*>(smem + kOffLPref);
    uint32_t* rbeg = reinterpret_cast<uint32_t*>(smem + kOffRBeg);    // this range's first posting per list
    uint32_t* ks = reinterpret_cast<uint32_t*>(smem + kOffKS);        // kept centroids' S rows (ord images, pitch 33)
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem + kOffBm);        // members of the range (pid bits)
    uint16_t* wpre = reinterpret_cast<uint16_t*>(smem + kOffWpre);    // members before each bitmap word
    uint16_t* mpid = reinterpret_cast<uint16_t*>(smem + kOffMPid);    // member rank -> pid offset in the range
    uint16_t* goff = reinterpret_cast<uint16_t*>(smem + kOffGOff);    // member rank -> kept-token count, then offset
    uint16_t* ulist = reinterpret_cast<uint16_t*>(smem + kOffUList);  // members with a kept token (this range)
    uint32_t* tile = reinterpret_cast<uint32_t*>(smem + kOffTile) + warp * 16 * 33;
    uint16_t* grp = reinterpret_cast<uint16_t*>(smem + kOffGrp);      // 33 x kept list of each kept token, by member
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + kOffHist);
    uint64_t* keys_used = side0 + 2 * a.c1cap;                        // keys of the members with a kept token
    const uint32_t W = a.range_w, R = a.range_n, WW = W / 32;
    // Every range must fit the shared-memory buffers: probed postings (an
    // upper bound on members) <= kMCap and kept postings <= kGCap; checked
    // from the range table, else stage 2 scans the candidates' codes.
    if (tid == 0) sh.maxp = 0, sh.maxk = 0;
    for (uint32_t s = tid; s < nprobed + min(kept_n, kKeptLists); s += kThreads) {
        const uint32_t c = s < nprobed ? probe[s] : kept[s - nprobed];
        lcent[s] = c;
        lstart[s] = __ldg(ix.ivf_offsets + c);
    }
    __syncthreads();
    {
        const uint32_t nk0 = min(kept_n, kKeptLists);
        for (uint32_t r = warp; r < R; r += kWarps) {
            uint32_t p = 0, k = 0;
            for (uint32_t s = lane; s < nprobed + nk0; s += 32) {
                const uint32_t* row = a.range_tab + uint64_t(lcent[s]) * (R + 1) + r;
                const uint32_t n = __ldg(row + 1) - __ldg(row);
                if (s < nprobed) p += n; else k += n;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o), k += __shfl_xor_sync(0xffffffffu, k, o);
            if (lane == 0) atomicMax(&sh.maxp, p), atomicMax(&sh.maxk, k);
        }
    }
    __syncthreads();
    const bool walk = kept_n <= kKeptLists && sh.kept_post <= kListsPerCandidate * uint64_t(sh.probed_post) &&
                      sh.maxp <= kMCap && sh.maxk <= kGCap;
    const uint32_t nk = walk ? kept_n : 0u;
    const uint32_t nl = nprobed + nk;
    for (uint32_t j = warp; j < nk; j += kWarps)
        ks[j * 33 + lane] = dev::ord_f32(__ldg(S + uint64_t(kept[j]) * kScoresPitch + lane));
    for (uint32_t b = tid; b < 2048; b += kThreads) hist[b] = 0;
    if (tid == 0) sh.nused = 0, sh.npos = 0;
    __syncthreads();
    stamp(a, qi, 1);

    // ---- B-E: candidate generation and stage 2, one pid range at a time.
    // Range r = pids [r W, (r + 1) W).  A sorted posting list's postings in
    // the range are one run, located by the index's range table.  In shared
    // memory: the range's C1 members (bitmap, compacted in id order), the
    // member each kept posting belongs to, grouped by member with a counting
    // sort, and per member with kept tokens the max of their centroids' S rows
    // per query token and the in-order sum: the stage-2 key.  One round trip
    // per range (probed and kept postings and the next range's run bounds
    // loaded together); nothing per query is N-sized, so hundreds of queries
    // in flight do not thrash L2.
    uint32_t n1 = 0;
    uint32_t tb[2] = {0, 0}, te[2] = {0, 0};  // run bounds of lists 2 tid, 2 tid + 1 in the current range
    auto load_bounds = [&](uint32_t r, uint32_t (&b)[2], uint32_t (&e)[2]) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            const uint32_t sidx = tid * 2 + x;
            b[x] = e[x] = 0;
            if (sidx < nl && r < R) {
                const uint32_t* row = a.range_tab + uint64_t(lcent[sidx]) * (R + 1) + r;
                b[x] = __ldg(row), e[x] = __ldg(row + 1);
            }
        }
    };
    load_bounds(0, tb, te);
    unsigned long long tacc[6] = {0, 0, 0, 0, 0, 0}, tprev = gtime();
    auto lap = [&](int k) {
        if (a.trace && tid == 0) {
            const unsigned long long t = gtime();
            tacc[k] += t - tprev;
            tprev = t;
        }
    };
    for (uint32_t r = 0; r < R; ++r) {
        // (1) run prefix over the lists; clear the range's member bitmap and counts
        for (uint32_t w = tid; w < WW; w += kThreads) bm[w] = 0u;
        for (uint32_t m = tid; m < kMCap; m += kThreads) goff[m] = 0;
        if (tid == 0) sh.ucount = 0;
        uint32_t tot;
        const uint32_t c0 = te[0] - tb[0], c1n = te[1] - tb[1];
        const uint32_t ex = block_excl_scan(c0 + c1n, sh.warp_tot, &tot);
        if (tid * 2 < nl) lpref[tid * 2] = ex, rbeg[tid * 2] = tb[0];
        if (tid * 2 + 1 < nl) lpref[tid * 2 + 1] = ex + c0, rbeg[tid * 2 + 1] = tb[1];
        if (tid == 0) lpref[nl] = tot;
        // flat posting index -> list, when the range's runs fit the map
        // (shares the stage-2 tile's space, free until step 5)
        const bool use_map = tot <= kMapCap;
        if (use_map) {
            uint16_t* map = reinterpret_cast<uint16_t*>(smem + kOffTile);
            for (uint32_t i = 0; i < c0; ++i) map[ex + i] = uint16_t(tid * 2);
            for (uint32_t i = 0; i < c1n; ++i) map[ex + c0 + i] = uint16_t(tid * 2 + 1);
        }
        __syncthreads();
        const uint32_t total_p = lpref[nprobed], total = lpref[nl];
        const uint32_t base_pid = r * W;
        lap(0);
        auto locate = [&](uint32_t f, uint32_t lo, uint32_t hi) -> uint64_t {  // (list << 40) | posting index
            if (use_map) {
                lo = reinterpret_cast<const uint16_t*>(smem + kOffTile)[f];
            } else {
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (lpref[mid] <= f) lo = mid; else hi = mid;
                }
            }
            return (uint64_t(lo) << 40) | (lstart[lo] + rbeg[lo] + (f - lpref[lo]));
        };
        // (2) the probed and the kept postings (<= kGCap = one register
        // chunk) of the range in one round
        uint32_t pp[kPer], kp[kPer], kl[kPer];
#pragma unroll
        for (int x = 0; x < int(kPer); ++x) {
            const uint32_t f = x * kThreads + tid;
            const uint64_t a1 = locate(f < total_p ? f : (total_p ? total_p - 1 : 0), 0, nprobed);
            pp[x] = total_p ? __ldg(ix.ivf_postings + (a1 & 0xFFFFFFFFFFull)) : 0u;
            const uint32_t g = total_p + f;
            const uint64_t a2 = locate(g < total ? g : (total > total_p ? total - 1 : 0), nprobed, nl > nprobed ? nl : nprobed + 1);
            kp[x] = total > total_p ? __ldg(ix.ivf_postings + (a2 & 0xFFFFFFFFFFull)) : 0u;
            kl[x] = uint32_t(a2 >> 40) - nprobed;
        }
        uint32_t nb[2], ne[2];
        load_bounds(r + 1, nb, ne);  // next range's runs, in flight with the postings
#pragma unroll
        for (int x = 0; x < int(kPer); ++x)
            if (x * kThreads + tid < total_p) {
                const uint32_t o = pp[x] - base_pid;
                atomicOr(bm + (o >> 5), 1u << (o & 31));
            }
        for (uint32_t f0 = kPer * kThreads; f0 < total_p; f0 += kPer * kThreads) {  // long ranges
            uint32_t q[kPer];
#pragma unroll
            for (int x = 0; x < int(kPer); ++x) {
                const uint32_t f = f0 + x * kThreads + tid;
                q[x] = __ldg(ix.ivf_postings + (locate(f < total_p ? f : total_p - 1, 0, nprobed) & 0xFFFFFFFFFFull));
            }
#pragma unroll
            for (int x = 0; x < int(kPer); ++x)
                if (f0 + x * kThreads + tid < total_p) {
                    const uint32_t o = q[x] - base_pid;
                    atomicOr(bm + (o >> 5), 1u << (o & 31));
                }
        }
        __syncthreads();
        lap(1);
        // (3) compaction: C1 positions in id order (pipeline.cpp:83's sort)
        uint32_t m_r;
        {
            constexpr uint32_t kPW = kRangeWords / kThreads;
            uint32_t v[kPW], mine = 0;
            const uint32_t w0 = tid * kPW;
#pragma unroll
            for (uint32_t j = 0; j < kPW; ++j) {
                v[j] = w0 + j < WW ? bm[w0 + j] : 0u;
                mine += __popc(v[j]);
            }
            uint32_t pos = block_excl_scan(mine, sh.warp_tot, &m_r);  // m_r <= probed postings <= kMCap
#pragma unroll
            for (uint32_t j = 0; j < kPW; ++j) {
                if (w0 + j < WW) wpre[w0 + j] = uint16_t(pos);  // <= 32 (W/32 - 1) < 65536
                uint32_t x = v[j];
                while (x) {
                    const uint32_t o = (w0 + j) * 32 + (__ffs(x) - 1);
                    if (walk) mpid[pos] = uint16_t(o);
                    else c1[n1 + pos] = base_pid + o;
                    ++pos;
                    x &= x - 1;
                }
            }
        }
        __syncthreads();
        lap(2);
        if (walk) {
            // (4) kept postings -> their member (counting sort by member rank)
            uint32_t rk[kPer], at[kPer];
#pragma unroll
            for (int x = 0; x < int(kPer); ++x) {
                rk[x] = 0xFFFFFFFFu;
                if (total_p + x * kThreads + tid < total) {
                    const uint32_t o = kp[x] - base_pid;
                    const uint32_t wv = bm[o >> 5];
                    if ((wv >> (o & 31)) & 1u) {
                        rk[x] = wpre[o >> 5] + __popc(wv & ((1u << (o & 31)) - 1u));
                        at[x] = atomicAdd(reinterpret_cast<unsigned int*>(goff + (rk[x] & ~1u)), 1u << (16 * (rk[x] & 1u)));
                        at[x] = (at[x] >> (16 * (rk[x] & 1u))) & 0xFFFFu;  // counts <= kGCap: no carry between halves
                    }
                }
            }
            __syncthreads();
            lap(3);
            {  // exclusive scan of the counts over the m_r members (in place)
                constexpr uint32_t kPM = kMCap / kThreads;
                uint32_t v[kPM], mine = 0;
#pragma unroll
                for (uint32_t j = 0; j < kPM; ++j) v[j] = goff[tid * kPM + j], mine += v[j];
                uint32_t gt;
                uint32_t run = block_excl_scan(mine, sh.warp_tot, &gt);
#pragma unroll
                for (uint32_t j = 0; j < kPM; ++j) goff[tid * kPM + j] = uint16_t(run), run += v[j];
                if (tid == 0) goff[kMCap] = uint16_t(gt);
            }
            __syncthreads();
#pragma unroll
            for (int x = 0; x < int(kPer); ++x)
                if (rk[x] != 0xFFFFFFFFu) grp[goff[rk[x]] + at[x]] = uint16_t(kl[x] * 33);
            __syncthreads();
            lap(4);
            // (5) members: stage-2 key = in-order sum over the query tokens of
            // the max over the member's kept tokens (pipeline.cpp:112-131), or 0.
            // Members without one get their zero key here; the others are
            // listed and scored a warp of 32 at a time, lane = member: the
            // max over its kept rows (two halves of 16 query tokens in
            // registers) and the in-order sum, all in the lane — no tile
            // transpose, and the 32 members' row loads proceed side by side
            // (lane = query token with members one after another was a chain
            // of dependent loads per member: ~2.4 of 5 ms per query)
            for (uint32_t m = tid; m < m_r; m += kThreads) {
                if (goff[m + 1] > goff[m]) ulist[atomicAdd(&sh.ucount, 1u)] = uint16_t(m);
                else keys[n1 + m] = dev::make_key(0.0f, base_pid + mpid[m]);
            }
            __syncthreads();
            const uint32_t nu = sh.ucount;
            uint32_t npos = 0;
            for (uint32_t u0 = warp * 32; u0 < nu; u0 += kWarps * 32) {
                const bool live = u0 + lane < nu;
                const uint32_t m = live ? ulist[u0 + lane] : 0u;
                const uint32_t gs = live ? goff[m] : 0u, ge = live ? goff[m + 1] : 0u;
                float t = 0.0f;
#pragma unroll
                for (uint32_t h = 0; h < 2; ++h) {
                    uint32_t mx[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) mx[j] = 0;
                    for (uint32_t g = gs; g < ge; ++g) {
                        const uint32_t* row = ks + grp[g] + 16 * h;
#pragma unroll
                        for (int j = 0; j < 16; ++j) mx[j] = max(mx[j], row[j]);
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (16 * h + j < rows) t = __fadd_rn(t, dev::unord_f32(mx[j]));
                }
                uint64_t key = 0;
                if (live) {
                    key = dev::make_key(t, base_pid + mpid[m]);
                    keys[n1 + m] = key;
                    atomicAdd(&hist[uint32_t(key >> 53)], 1u);
                    npos += t > 0.0f;
                }
                const uint32_t lb = __ballot_sync(0xffffffffu, live);
                uint32_t ub0 = 0;
                if (lane == 0 && lb) ub0 = atomicAdd(&sh.nused, uint32_t(__popc(lb)));
                ub0 = __shfl_sync(0xffffffffu, ub0, 0);
                if (live) keys_used[ub0 + __popc(lb & ((1u << lane) - 1u))] = key;
            }
            if (npos) atomicAdd(&sh.npos, npos);
        }
        n1 += m_r;
        tb[0] = nb[0], tb[1] = nb[1], te[0] = ne[0], te[1] = ne[1];
        __syncthreads();
        lap(5);
    }
    if (a.trace && tid == 0) {  // slots 11-14: bounds+prefix, postings, compaction+count, scan+scatter+score
        a.trace[uint64_t(qi) * 16 + 11] = tacc[0];
        a.trace[uint64_t(qi) * 16 + 12] = tacc[1];
        a.trace[uint64_t(qi) * 16 + 13] = tacc[2] + tacc[3];
        a.trace[uint64_t(qi) * 16 + 14] = tacc[4] + tacc[5];
    }
    stamp(a, qi, 15);
    __threadfence();
    __syncthreads();
    const uint32_t nused = sh.nused;
    stamp(a, qi, 2);
    if (n1 == 0) {  // pipeline.cpp:245-248: empty result
        if (tid == 0) {
            a.out_n[qi] = 0;
            if (a.counters) {
                uint64_t* cn = a.counters + uint64_t(qi) * 4;
                cn[0] = cn[1] = cn[2] = cn[3] = 0;
            }
        }
        return;
    }
    uint32_t nsel2 = n1;
    const uint64_t* sel_in = keys;
    if (walk) {
        // every key of the top ndocs has a positive score when enough members
        // do (a zero-score key, kept token or not, ranks below them): select
        // among the members with a kept token only; else over every member
        if (sh.npos < min(a.ndocs, n1)) {
            if (tid == 0) hist[dev::ord_f32(0.0f) >> 21] += n1 - nused;
        } else {
            nsel2 = nused;
            sel_in = keys_used;
        }
    } else {
        // code scan: warp per candidate over its codes (masked)
        for (uint32_t i = warp; i < n1; i += kWarps) {
            const uint32_t pid = __ldcg(c1 + i);
            uint32_t usedn;
            const float total = score_passage(ix.codes, __ldg(ix.offsets + pid), __ldg(ix.doclens + pid), S, rows, keep,
                                              true, &usedn);
            if (lane == 0) {
                const uint64_t key = dev::make_key(total, pid);
                keys[i] = key;
                atomicAdd(&hist[uint32_t(key >> 53)], 1u);
            }
        }
    }
    __threadfence();
    __syncthreads();
    stamp(a, qi, 3);
    const uint32_t n2 = cta_select(sel_in, nsel2, a.ndocs, sel2, side0, side1, hist, sh, true);
    stamp(a, qi, 6);

    // ---- F: stage 3 over the survivors
    // F0: (offset, len) of every survivor
    uint64_t* m_off = side0;
    uint32_t* m_len = reinterpret_cast<uint32_t*>(side1);
    for (uint32_t i0 = 0; i0 < n2; i0 += 4 * kThreads) {
        uint32_t pid[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const uint32_t i = i0 + x * kThreads + tid < n2 ? i0 + x * kThreads + tid : n2 - 1;
            pid[x] = dev::key_id(__ldcg(sel2 + i));
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const uint32_t i = i0 + x * kThreads + tid;
            const uint64_t off = __ldg(ix.offsets + pid[x]);
            const uint32_t len = __ldg(ix.doclens + pid[x]);
            if (i < n2) m_off[i] = off, m_len[i] = len;
        }
    }
    __threadfence();
    __syncthreads();
    // F1: warp w walks the concatenated tokens of its passages w, w + 8, ...
    // (batches of 32), 32 stream positions per step with all 32 S-row
    // gathers in flight; the running max (lane = query token) restarts at a
    // passage start and goes to the passage's row of acc when it ends
    for (uint32_t jb = 0;; jb += 32) {
        const uint32_t il = warp + kWarps * (jb + lane);
        const bool has = il < n2;
        if (!__any_sync(0xffffffffu, has)) break;
        const uint64_t poff = has ? __ldcg(m_off + il) : 0;
        const uint32_t plen = has ? __ldcg(m_len + il) : 0;
        uint32_t incl = plen;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31), excl = incl - plen;
        auto locate = [&](uint32_t s, uint32_t& p, uint32_t& code) {
            uint32_t lo = 0;
#pragma unroll
            for (uint32_t st = 16; st > 0; st >>= 1) {
                const uint32_t cand = lo + st;
                const uint32_t e = __shfl_sync(0xffffffffu, excl, cand & 31);
                if (cand < 32 && e <= s) lo = cand;
            }
            p = lo;
            const uint64_t o = __shfl_sync(0xffffffffu, poff, lo);
            const uint32_t e = __shfl_sync(0xffffffffu, excl, lo);
            code = __ldg(ix.codes + o + (s < total ? s - e : 0u));
        };
        uint32_t p_cur = 0, code_cur = 0;
        if (total) locate(lane < total ? lane : total - 1, p_cur, code_cur);
        float accv = -INFINITY;
        int cur = -1;
        for (uint32_t s0 = 0; s0 < total; s0 += 32) {
            const uint32_t nv = total - s0 < 32 ? total - s0 : 32u;
            float row[32];
#pragma unroll
            for (int v = 0; v < 32; ++v) {
                const uint32_t c = __shfl_sync(0xffffffffu, code_cur, uint32_t(v) < nv ? v : nv - 1);
                row[v] = __ldg(S + uint64_t(c) * kScoresPitch + lane);
            }
            const uint32_t p_this = p_cur;
            if (s0 + 32 < total) {  // next step's positions and codes, in flight with the gathers
                const uint32_t s = s0 + 32 + lane;
                locate(s < total ? s : total - 1, p_cur, code_cur);
            }
#pragma unroll
            for (int v = 0; v < 32; ++v) {
                if (uint32_t(v) >= nv) break;
                const int pv = int(__shfl_sync(0xffffffffu, p_this, v));
                if (pv != cur) {
                    if (cur >= 0)
                        acc[uint64_t(warp + kWarps * (jb + uint32_t(cur))) * 32 + lane] = __float_as_uint(accv);
                    accv = -INFINITY;
                    cur = pv;
                }
                accv = dev::max_gt(accv, row[v]);
            }
        }
        if (cur >= 0) acc[uint64_t(warp + kWarps * (jb + uint32_t(cur))) * 32 + lane] = __float_as_uint(accv);
    }
    __threadfence();
    __syncthreads();
    // F2: keys (in-order sum over the query tokens), rows re-zeroed
    for (uint32_t i = tid; i < n2; i += kThreads) {
        uint4 r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = __ldcg(reinterpret_cast<const uint4*>(acc + uint64_t(i) * 32) + q);
        const uint32_t len = __ldcg(m_len + i);
        const uint32_t pid = dev::key_id(__ldcg(sel2 + i));
        float total = 0.0f;
        if (len) {
            const uint32_t* rv = reinterpret_cast<const uint32_t*>(r);
#pragma unroll
            for (int q = 0; q < 32; ++q)
                if (uint32_t(q) < rows) total = __fadd_rn(total, __uint_as_float(rv[q]));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) reinterpret_cast<uint4*>(acc + uint64_t(i) * 32)[q] = make_uint4(0, 0, 0, 0);
        keys[i] = dev::make_key(total, pid);
    }
    __threadfence();
    __syncthreads();
    stamp(a, qi, 7);
    const uint32_t n3 = cta_select(keys, n2, a.n3, sel3, side0, side1, hist, sh, false);
    stamp(a, qi, 8);

    // ---- G: stage 4
    if (a.s4_tensor) {
        stage4_tensor<NB>(ix, a, Q, S, rows, n3, sel3, side0, reinterpret_cast<uint32_t*>(side1), smem);
    } else {
    // exact decompression + MaxSim of the finalists
    float* qs = reinterpret_cast<float*>(smem + kOffQ);
    float* vb = reinterpret_cast<float*>(smem + kOffV) + warp * (kTok * 128);
    uint64_t* k4 = reinterpret_cast<uint64_t*>(smem + kOffK4);
    uint64_t* f_off = side0;
    uint32_t* f_len = reinterpret_cast<uint32_t*>(side1);
    for (uint32_t e = tid; e < 32 * 32; e += kThreads) {  // 32 rows x 32 float4
        const uint32_t r = e >> 5, d4 = e & 31;
        const float4 v = r < rows ? __ldg(reinterpret_cast<const float4*>(Q + r * 128) + d4) : make_float4(0, 0, 0, 0);
        *reinterpret_cast<float4*>(qs + r * kQPitch + 4 * d4) = v;
    }
    for (uint32_t i = tid; i < n3; i += kThreads) {
        const uint32_t pid = dev::key_id(__ldcg(sel3 + i));
        f_off[i] = __ldg(ix.offsets + pid);
        f_len[i] = __ldg(ix.doclens + pid);
    }
    __threadfence();
    __syncthreads();
    constexpr uint32_t kBpt = NB * 128 / 8;  // residual bytes per token
    constexpr uint32_t kMask = (1u << NB) - 1;
    const float* qrow = qs + lane * kQPitch;
    float wts[1 << NB];
#pragma unroll
    for (int j = 0; j < (1 << NB); ++j) wts[j] = ix.weights[j];
    // software pipeline over groups of kTok tokens: while group g is
    // decoded and scored, group g + 1's centroid rows / residuals / norms and
    // group g + 2's codes are in flight
    struct Tok {
        float4 c;
        uint32_t rb;
        float inv;
    };
    auto load_codes = [&](uint64_t off, uint32_t len, uint32_t t0, uint32_t (&code)[kTok]) {
#pragma unroll
        for (int u = 0; u < int(kTok); ++u) code[u] = __ldg(ix.codes + off + min(t0 + u, len - 1));
    };
    auto load_data = [&](uint64_t off, uint32_t len, uint32_t t0, const uint32_t (&code)[kTok], Tok (&d)[kTok]) {
#pragma unroll
        for (int u = 0; u < int(kTok); ++u) {
            const uint64_t tok = off + min(t0 + u, len - 1);
            d[u].c = __ldg(reinterpret_cast<const float4*>(ix.centroids + uint64_t(code[u]) * 128) + lane);
            d[u].inv = __ldg(ix.tok_inv + tok);
            if constexpr (NB == 1) d[u].rb = (__ldg(ix.residuals + tok * kBpt + (lane >> 1)) >> ((lane & 1) * 4)) & 0xFu;
            else if constexpr (NB == 2) d[u].rb = __ldg(ix.residuals + tok * kBpt + lane);
            else d[u].rb = __ldg(reinterpret_cast<const uint16_t*>(ix.residuals + tok * kBpt) + lane);
        }
    };
    for (uint32_t f = warp; f < n3; f += kWarps) {
        const uint64_t off = __ldcg(f_off + f);
        const uint32_t len = __ldcg(f_len + f);
        float best = -INFINITY;
        uint32_t cn[kTok], cnn[kTok];
        Tok cur[kTok], nxt[kTok];
        load_codes(off, len, 0, cn);
        load_data(off, len, 0, cn, cur);
        load_codes(off, len, kTok, cn);
        for (uint32_t t0 = 0; t0 < len; t0 += kTok) {
            if (t0 + kTok < len) {
                load_data(off, len, t0 + kTok, cn, nxt);
                load_codes(off, len, t0 + 2 * kTok, cnn);
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < int(kTok); ++u) {
                float4 v;  // v = (C + w[bucket]) * inv (residual_codec.cpp:113-130)
                v.x = __fmul_rn(__fadd_rn(cur[u].c.x, wts[(cur[u].rb >> (0 * NB)) & kMask]), cur[u].inv);
                v.y = __fmul_rn(__fadd_rn(cur[u].c.y, wts[(cur[u].rb >> (1 * NB)) & kMask]), cur[u].inv);
                v.z = __fmul_rn(__fadd_rn(cur[u].c.z, wts[(cur[u].rb >> (2 * NB)) & kMask]), cur[u].inv);
                v.w = __fmul_rn(__fadd_rn(cur[u].c.w, wts[(cur[u].rb >> (3 * NB)) & kMask]), cur[u].inv);
                reinterpret_cast<float4*>(vb + u * 128)[lane] = v;
            }
            __syncwarp();
            // lane = query token: kTok independent in-order dot chains
            float sdot[kTok];
#pragma unroll
            for (int u = 0; u < int(kTok); ++u) sdot[u] = 0.0f;
#pragma unroll 4
            for (uint32_t d4 = 0; d4 < 32; ++d4) {
                const float4 x = *reinterpret_cast<const float4*>(qrow + 4 * d4);
#pragma unroll
                for (int u = 0; u < int(kTok); ++u) {
                    const float4 y = reinterpret_cast<const float4*>(vb + u * 128)[d4];
                    const float2 p01 = mul2(make_float2(x.x, x.y), make_float2(y.x, y.y));
                    const float2 p23 = mul2(make_float2(x.z, x.w), make_float2(y.z, y.w));
                    sdot[u] = __fadd_rn(sdot[u], p01.x);
                    sdot[u] = __fadd_rn(sdot[u], p01.y);
                    sdot[u] = __fadd_rn(sdot[u], p23.x);
                    sdot[u] = __fadd_rn(sdot[u], p23.y);
                }
            }
#pragma unroll
            for (int u = 0; u < int(kTok); ++u)
                if (t0 + u < len) best = (t0 + u == 0) ? sdot[u] : dev::max_gt(best, sdot[u]);
#pragma unroll
            for (int u = 0; u < int(kTok); ++u) cur[u] = nxt[u], cn[u] = cnn[u];
        }
        float total = 0.0f;
        for (uint32_t j = 0; j < rows; ++j) total = __fadd_rn(total, __shfl_sync(0xffffffffu, best, j));
        if (lane == 0) k4[f] = dev::make_key(total, dev::key_id(__ldcg(sel3 + f)));
    }
    }
    __syncthreads();
    stamp(a, qi, 9);
    uint64_t* k4 = reinterpret_cast<uint64_t*>(smem + kOffK4);
    // ---- H: top-k (bitonic sort, descending)
    uint32_t np2 = 1;
    while (np2 < n3) np2 <<= 1;
    for (uint32_t f = n3 + tid; f < np2; f += kThreads) k4[f] = 0;
    __syncthreads();
    for (uint32_t size = 2; size <= np2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < np2 / 2; i += kThreads) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const uint64_t x = k4[lo], y = k4[hi];
                if ((x < y) == desc) k4[lo] = y, k4[hi] = x;
            }
            __syncthreads();
        }
    }
    const uint32_t nout = n3 < a.k ? n3 : a.k;
    for (uint32_t j = tid; j < nout; j += kThreads) {
        const uint64_t key = k4[j];
        a.out_pids[uint64_t(qi) * a.k + j] = dev::key_id(key) + a.pid_base;
        a.out_scores[uint64_t(qi) * a.k + j] = dev::key_score(key);
    }
    if (tid == 0) {
        a.out_n[qi] = nout;
        if (a.counters) {
            uint64_t* cn = a.counters + uint64_t(qi) * 4;
            cn[0] = n1, cn[1] = n2, cn[2] = n3, cn[3] = nout;
        }
    }
    stamp(a, qi, 10);
}

// tab[c][r] = offset in c's sorted posting list of its first posting >= r W
// (binary search; index-load time, once per index)
__global__ void range_table_kernel(const uint64_t* __restrict__ ivf_offsets, const uint32_t* __restrict__ postings,
                                   uint64_t K, uint32_t W, uint32_t R, uint32_t* __restrict__ tab) {
    const uint64_t n = K * uint64_t(R + 1);
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = e / (R + 1), r = e % (R + 1);
        const uint64_t b = ivf_offsets[c], end = ivf_offsets[c + 1];
        const uint64_t key = r * uint64_t(W);
        uint64_t lo = b, hi = end;  // first index with postings[i] >= key
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (uint64_t(postings[mid]) < key) lo = mid + 1; else hi = mid;
        }
        tab[e] = uint32_t(lo - b);
    }
}

template <int NP>
void launch_np(const IndexView& ix, const launch::WaveArgs& a, uint32_t nq, cudaStream_t st) {
    auto k = ix.nbits == 1 ? wave_worker_kernel<NP, 1> : ix.nbits == 2 ? wave_worker_kernel<NP, 2>
                                                                       : wave_worker_kernel<NP, 4>;
    static launch::PerDeviceOnce configured;
    if (configured.first()) {
        cudaFuncSetAttribute(wave_worker_kernel<NP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(wave_worker_kernel<NP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(wave_worker_kernel<NP, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    }
    ::plaid::launch::pdl(k, nq, kThreads, kSmemBytes, st, ix, a);
    launch::count_launch();
}

}  // namespace

namespace launch {

void wave_worker(const IndexView& ix, const WaveArgs& a, uint32_t nq, uint32_t np_stride, cudaStream_t st) {
    if (nq == 0) return;
    switch (np_stride) {
        case 1: launch_np<1>(ix, a, nq, st); break;
        case 2: launch_np<2>(ix, a, nq, st); break;
        case 4: launch_np<4>(ix, a, nq, st); break;
        case 8: launch_np<8>(ix, a, nq, st); break;
        default: fail_cuda_driver(1, "wave worker supports np buckets <= 8");
    }
}

uint32_t wave_worker_ctas_per_sm(uint32_t nbits) {
    auto k = nbits == 1 ? wave_worker_kernel<8, 1> : nbits == 2 ? wave_worker_kernel<8, 2> : wave_worker_kernel<8, 4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kThreads, kSmemBytes) != cudaSuccess || n < 1) n = 1;
    return uint32_t(n);
}

void wave_range_table(const IndexView& ix, uint32_t W, uint32_t R, uint32_t* d_tab, cudaStream_t st) {
    const uint64_t n = ix.K * uint64_t(R + 1);
    const uint32_t blocks = uint32_t(std::min<uint64_t>((n + 255) / 256, 1u << 20));
    range_table_kernel<<<blocks, 256, 0, st>>>(ix.ivf_offsets, ix.ivf_postings, ix.K, W, R, d_tab);
    count_launch();
}

}  // namespace launch
}  // namespace plaid
