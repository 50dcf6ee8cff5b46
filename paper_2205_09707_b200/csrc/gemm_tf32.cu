// gemm_tf32.cu — stage-1 S_cq = C . Q^T on the 5th-gen tensor cores (tcgen05),
// the production score path (PLAID_SCORES_TENSOR).  Replaces the reference's
// scalar compute_centroid_scores (pipeline.cpp:26-50) and fuses the two
// consumers of S that follow it: the per-token top-nprobe selection
// (pipeline.cpp:52-88) and the t_cs keep mask of centroid pruning
// (pipeline.cpp:90-110).
//
// Precision: 3xTF32.  Each fp32 operand is split into hi = x with the low 13
// mantissa bits cleared and lo = x - hi (the tensor core truncates fp32
// operands to tf32, tools/tf32_round.cu: C_hi is the raw row, and C_lo is
// truncated in turn — Q_lo is rounded, it is built once per query), and
// S = C_hi.Q_hi + C_hi.Q_lo + C_lo.Q_hi is accumulated in fp32 in TMEM: ~2e-6
// absolute on unit-vector dots (tests/test_gpu_parity.py), while HBM traffic
// stays one fp32 read of C.
//
// Structure (persistent, one CTA per SM, 16 warps):
//   warp 0      TMA producer: 128-centroid x 32-dim fp32 boxes (16 KB,
//               SWIZZLE_128B) into a 9-stage ring (144 KB in flight);
//   warps 4-7   converters: thread = centroid row; read the row's 32 floats
//               of a landed box (conflict-free LDS.128 through the swizzle),
//               release the slot, split, and write C_hi / C_lo straight into
//               TMEM (tcgen05.st: lane = row, column = k) — the MMA A operand;
//   warp 1      MMA issuer (one thread): per 8-dim step one M=128 N=64 MMA
//               C_hi . [Q_hi | Q_lo] and one N=32 MMA C_lo . Q_hi into the
//               same accumulator, B = Q from shared memory (8 KB per chunk);
//   warps 8-15  epilogue, two groups of four taking alternate tiles (group g
//               owns accumulator g): tcgen05.ld of the 64 accumulator
//               columns, S = hi + lo products, the keep bit (row max >= t_cs
//               -> one ballot -> one 32-bit word), a 32x32 transpose through
//               shared memory, then lane = token: the S row stores (one
//               coalesced 128-byte row per centroid) and the per-token
//               top-nprobe (score, id) list, where a float threshold plus
//               CTA- and grid-wide bounds make inserts rare;
//   warps 2-3   idle.
// Shared-memory traffic per 128-centroid tile is ~200 KB (TMA write, converter
// read, MMA B reads, transpose): ~0.8 us at 128 B/clk, under the ~1.5 us the
// tile takes to stream from HBM when all 148 SMs pull at once.  (The first
// design, with C as the smem B operand split in shared memory, moved ~384 KB
// per tile and was shared-memory bound at ~2 us per tile.)
// TMEM: [0,128) two 64-column accumulators; [128,512) six operand slots of
// 32 C_hi + 32 C_lo columns.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "device.cuh"
#include "kernels.cuh"

namespace plaid {
namespace {

constexpr uint32_t kChunkBytes = 128 * 128;  // one TMA box: 32 centroids x 128 fp32 (16 KB contiguous in HBM)
constexpr int kThreads = 512;
constexpr int kEpiWarps = 8;                 // warps 8..15
constexpr uint32_t kTmemCols = 512;
constexpr int kDim = 128;
constexpr int kChunks = kDim / 32;

// kind::tf32 instruction descriptors: D f32, A/B tf32, both K-major, M=128.
constexpr uint32_t idesc_tf32(uint32_t n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

// Per-batch-width layout: QB queries share one pass over C.  B operand rows
// [0, 32 QB) = Q_hi of query r / 32, [32 QB, 64 QB) = Q_lo; accumulator
// columns [32 qi, +32) = C_hi.Q_hi + C_lo.Q_hi of query qi and
// [32 QB + 32 qi, +32) = C_hi.Q_lo of query qi.
template <int QB>
struct TfCfg {
    // TMA ring depth.  Box gb (tile gb / 4, lane quarter gb % 4) shares its
    // slot with box gb - kRaw; a converter warp can reach box gb once the MMA
    // has consumed tile gb / 4 - 2, so box gb - kRaw must belong to that tile
    // or earlier (else a parity wait two phases behind passes on a stale
    // box): kRaw = 8 (same quarter) or kRaw >= 9.  7 is NOT safe.
    static constexpr int kRaw = QB == 1 ? 9 : 8;
    static constexpr int kOps = QB == 1 ? 6 : 4;        // TMEM operand slots (64 columns each)
    static constexpr uint32_t kQChunkBytes = 64 * QB * 128;
    static constexpr uint32_t kAccCols = 64 * QB;       // per accumulator (two, double-buffered)
    static constexpr uint32_t kOpsCol0 = 2 * kAccCols;  // first operand-slot column
    static_assert(kOpsCol0 + 64 * kOps <= kTmemCols, "TMEM budget");
    // shared-memory carve-up (offsets from a 1024-B aligned base)
    static constexpr uint32_t kOffRaw = 0;
    static constexpr uint32_t kOffQ = kOffRaw + kRaw * kChunkBytes;
    static constexpr uint32_t kOffTr = kOffQ + kChunks * kQChunkBytes;  // 8 warps x 32 x 33 floats
    static constexpr uint32_t kOffBar = kOffTr + kEpiWarps * 32 * 33 * 4;
    static constexpr uint32_t kNumBars = 2 * kRaw + 2 * kOps + 4;
    static constexpr uint32_t kOffMisc = kOffBar + kNumBars * 8;  // tmem slot (16 B) + CTA bounds (128 B per query)
    static constexpr uint32_t kSmemBytes = kOffMisc + 16 + 128 * QB + 1024;  // + alignment slack
    static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
    static constexpr uint32_t kIdescAll = idesc_tf32(64 * QB);  // C_hi . [Q_hi | Q_lo] of every query
    static constexpr uint32_t kIdescHi = idesc_tf32(32 * QB);   // C_lo . Q_hi of every query
};

// Debug timeline (PLAID_TF32_DBG=16): globaltimer stamps of CTA 0's pipeline
// events and every CTA's begin/end (read back with plaid_debug_tf32_trace).
// Pipeline experiments (results wrong): dbg & 1 skips the MMAs, & 2 the S
// stores, & 4 the TMEM operand stores, & 8 the converters' reads.
__device__ unsigned long long g_tf32_trace[8 * 256];
__device__ unsigned long long g_tf32_cta[2 * 256];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_stamp(uint32_t dbg, int slot, uint32_t i) {
    if ((dbg & 16) && blockIdx.x == 0 && i < 256) g_tf32_trace[slot * 256 + i] = gtime();
}
__device__ __forceinline__ void cta_stamp(uint32_t dbg, int which) {
    if ((dbg & 16) && threadIdx.x == 0 && blockIdx.x < 256) g_tf32_cta[which * 256 + blockIdx.x] = gtime();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// suspend-time hint: a waiting warp sleeps until the phase completes instead
// of re-polling (the polls were 16% of the issued instructions)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(0x100000)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (SM100 layout:
// start>>4 @0, LBO>>4 @16 (unused for swizzled K-major), SBO>>4 @32 = 1024 B
// between 8-row groups, version 1 @46, layout 2 = SWIZZLE_128B @61).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr) {
    uint64_t d = uint64_t((addr >> 4) & 0x3FFFu);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

// One 32-dim chunk of a tile, issued by the whole (converged) warp with the
// elected lane predicated inside a single asm block: per 8-dim step
// D[:, 0:32QB] += C_hi.Q_hi, D[:, 32QB:64QB] += C_hi.Q_lo (idesc_all) and
// D[:, 0:32QB] += C_lo.Q_hi (idesc_hi), then a commit to `bar`.  Issued from a
// `lane == 0` branch instead, every MMA was wrapped in its own waterfall loop
// (ELECT / R2UR.BROADCAST / BRA.U.ANY) and the issuing warp, not the tensor
// core, set the pace: ~0.45 us per chunk against ~0.2 us of MMA work
// (tools/tf32_timeline.py).  Descriptor steps: +32 bytes of K = +2 in the
// smem descriptor's address field, +8 TMEM columns.
__device__ __forceinline__ void mma_chunk_tf32(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t b, uint32_t idesc_all,
                                               uint32_t idesc_hi, uint32_t accumulate, uint32_t bar) {
    asm volatile(
        "{\n\t"
        ".reg .pred e, pa, pt;\n\t"
        ".reg .b32 rx, h1, h2, h3, l1, l2, l3;\n\t"
        ".reg .b64 b1, b2, b3;\n\t"
        "elect.sync rx|e, 0xffffffff;\n\t"
        "setp.ne.b32 pa, %6, 0;\n\t"
        "setp.eq.b32 pt, %6, %6;\n\t"
        "add.s64 b1, %3, 2;\n\t"
        "add.s64 b2, %3, 4;\n\t"
        "add.s64 b3, %3, 6;\n\t"
        "add.u32 h1, %1, 8;\n\t"
        "add.u32 h2, %1, 16;\n\t"
        "add.u32 h3, %1, 24;\n\t"
        "add.u32 l1, %2, 8;\n\t"
        "add.u32 l2, %2, 16;\n\t"
        "add.u32 l3, %2, 24;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %4, pa;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h1], b1, %4, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [l1], b1, %5, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h2], b2, %4, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [l2], b2, %5, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [h3], b3, %4, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [l3], b3, %5, pt;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t"
        "}" ::"r"(d),
        "r"(ahi), "r"(alo), "l"(b), "r"(idesc_all), "r"(idesc_hi), "r"(accumulate), "r"(bar)
        : "memory");
}

// tcgen05.commit by the elected lane of a converged warp.
__device__ __forceinline__ void mma_commit_warp(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
        "elect.sync rx|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}


// 32 consecutive TMEM columns of this warp's 32 lanes -> r[0..31] (no wait).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// r[0..31] -> 32 consecutive TMEM columns of this warp's 32 lanes.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ uint32_t split_hi(uint32_t x) { return x & 0xFFFFE000u; }
__device__ __forceinline__ uint32_t lo_trunc(uint32_t x) {
    return __float_as_uint(__fsub_rn(__uint_as_float(x), __uint_as_float(split_hi(x))));
}

// x - trunc_tf32(x) rounded to the nearest tf32 (an unrounded lo would be
// truncated again by the tensor core and bias every dot product downwards)
__device__ __forceinline__ uint32_t split_lo(uint32_t x) {
    const float lo = __fsub_rn(__uint_as_float(x), __uint_as_float(split_hi(x)));
    return (__float_as_uint(lo) + 0x1000u) & 0xFFFFE000u;
}

template <int NP, int QB>
__global__ void __launch_bounds__(kThreads, 1)
scores_tf32_kernel(const __grid_constant__ CUtensorMap cmap, uint64_t K, const __grid_constant__ TfOut out,
                   uint32_t rows, float t_cs, uint32_t dbg) {
    using Cf = TfCfg<QB>;
    constexpr int kRaw = Cf::kRaw, kOps = Cf::kOps;
    constexpr uint32_t kOffRaw = Cf::kOffRaw, kOffQ = Cf::kOffQ, kOffTr = Cf::kOffTr, kOffBar = Cf::kOffBar,
                       kOffMisc = Cf::kOffMisc, kQChunkBytes = Cf::kQChunkBytes, kAccCols = Cf::kAccCols,
                       kOpsCol0 = Cf::kOpsCol0;
    // No griddepcontrol.wait yet: C is index data no earlier kernel writes,
    // so the TMA producer starts streaming it while the previous kernel (the
    // query prologue, which triggers its dependents at once) still runs;
    // every other warp waits before it touches Q, the bounds or the outputs.
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t base = smem_u32(smem);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = base + kOffBar;
    auto raw_full = [&](int s) { return bar0 + 8u * s; };
    auto raw_empty = [&](int s) { return bar0 + 8u * (kRaw + s); };
    auto ops_full = [&](int s) { return bar0 + 8u * (2 * kRaw + s); };
    auto ops_empty = [&](int s) { return bar0 + 8u * (2 * kRaw + kOps + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * kRaw + 2 * kOps + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * kRaw + 2 * kOps + 2 + a); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffMisc);
    // CTA-wide per-token bound per query, cthr[32 qi + token] (ordered float bits, 0 = none)
    volatile uint32_t* cthr = reinterpret_cast<volatile uint32_t*>(smem + kOffMisc + 16);

    const uint64_t ntiles = (K + 127) / 128;
    cta_stamp(dbg, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRaw; ++s) {
            mbar_init(raw_full(s), 1);
            mbar_init(raw_empty(s), 1);  // the converter warp of the box's lane quarter
        }
        for (int s = 0; s < kOps; ++s) {
            mbar_init(ops_full(s), 4);
            mbar_init(ops_empty(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), kEpiWarps / 2);  // the 4 warps of group a
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&cmap)) : "memory");
    }
    // box gb of this CTA = tile blockIdx.x + (gb / 4) * gridDim.x, lane quarter gb % 4
    const uint64_t my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint32_t nboxes = uint32_t(my_tiles * 4);
    auto issue_box = [&](uint32_t g) {
        const int s = g % kRaw;
        mbar_wait(raw_empty(s), ((g / kRaw) & 1) ^ 1);
        trace_stamp(dbg, 0, g);
        mbar_expect_tx(raw_full(s), kChunkBytes);
        const uint64_t t = blockIdx.x + uint64_t(g / 4) * gridDim.x;
        tma_load_3d(base + kOffRaw + s * kChunkBytes, &cmap, 0, int(t * 128 + (g % 4) * 32), 0, raw_full(s));
    };
    // the ring's first fill goes out before anything waits on earlier kernels
    const uint32_t pre = nboxes < uint32_t(kRaw) ? nboxes : uint32_t(kRaw);
    if (threadIdx.x == 0)
        for (uint32_t g = 0; g < pre; ++g) issue_box(g);
    if (warp != 0) dev::pdl_wait();
    if (threadIdx.x < 32 * QB) cthr[threadIdx.x] = 0;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // B operand [Q_hi of every query; Q_lo of every query] (row n < 32 QB:
    // Q_hi of query n / 32, token n % 32, else Q_lo; zero rows past `rows`),
    // SWIZZLE_128B K-major: row n, 16-byte granule j of chunk kc at
    // kc * kQChunkBytes + n*128 + ((j ^ (n & 7)) << 4)
    for (uint32_t e = threadIdx.x - 32; warp != 0 && e < 64 * QB * (kDim / 4); e += kThreads - 32) {
        const uint32_t n = e / (kDim / 4), g = e % (kDim / 4);
        const uint32_t kc = g / 8, j = g % 8, tok = n & 31, qi = (n % (32 * QB)) / 32;
        const uint4 v = tok < rows ? reinterpret_cast<const uint4*>(out.Q[qi] + uint64_t(tok) * kDim)[g]
                                   : make_uint4(0, 0, 0, 0);
        const uint32_t off = kc * kQChunkBytes + n * 128 + ((j ^ (n & 7)) << 4);
        *reinterpret_cast<uint4*>(smem + kOffQ + off) =
            n < 32 * QB ? make_uint4(split_hi(v.x), split_hi(v.y), split_hi(v.z), split_hi(v.w))
                        : make_uint4(split_lo(v.x), split_lo(v.y), split_lo(v.z), split_lo(v.w));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer: box (t, w) = centroids [128 t + 32 w,
        // +32), all 128 dims: 16 KB contiguous in HBM, landing as
        // [chunk][centroid][32 fp32]; the first `pre` boxes went out above
        if (lane == 0)
            for (uint32_t g = pre; g < nboxes; ++g) issue_box(g);
    } else if (warp == 1) {
        // ---------------- MMA issuer
        uint32_t g = 0, lt = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
            const uint32_t acc = lt & 1;
            mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d = tmem_base + acc * kAccCols;
            for (int kc = 0; kc < kChunks; ++kc, ++g) {
                const int s = g % kOps;
                mbar_wait(ops_full(s), (g / kOps) & 1);
                if (lane == 0) trace_stamp(dbg, 4, g);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (!(dbg & 1)) {
                    const uint32_t ahi = tmem_base + kOpsCol0 + s * 64, alo = ahi + 32;
                    const uint32_t bq = base + kOffQ + kc * kQChunkBytes;
                    mma_chunk_tf32(d, ahi, alo, umma_desc(bq), Cf::kIdescAll, Cf::kIdescHi, uint32_t(kc), ops_empty(s));
                    if (kc == kChunks - 1) mma_commit_warp(tfull_bar(acc));
                } else if (lane == 0) {  // dbg & 1: no MMAs (pipeline experiment)
                    mbar_arrive(ops_empty(s));
                    if (kc == kChunks - 1) mbar_arrive(tfull_bar(acc));
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- converters: warp = lane quarter q, thread = centroid
        // row 32 q + lane; the warp owns box (t, q) of every tile
        const uint32_t q = warp & 3;
        const uint32_t lane_off = (q * 32) << 16;
        uint32_t go = 0, lt = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
            const uint32_t gb = lt * 4 + q;
            const int s = gb % kRaw;
            mbar_wait(raw_full(s), (gb / kRaw) & 1);
            if (warp == 4 && lane == 0) trace_stamp(dbg, 1, lt * 4);
            if (dbg & 8) {  // experiment: pure TMA stream (box released unread, no MMA input)
                __syncwarp();
                if (lane == 0) mbar_arrive(raw_empty(s));
                for (int kc = 0; kc < kChunks; ++kc, ++go) {
                    const int o = go % kOps;
                    mbar_wait(ops_empty(o), ((go / kOps) & 1) ^ 1);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(ops_full(o));
                }
                continue;
            }
            for (int kc = 0; kc < kChunks; ++kc, ++go) {
                const int o = go % kOps;
                // the row's 8 granules of chunk kc, un-swizzled: granule j at (j ^ (lane & 7))
                const uint4* src =
                    reinterpret_cast<const uint4*>(smem + kOffRaw + s * kChunkBytes + (kc * 32 + lane) * 128);
                // A_hi = the raw fp32 row (the tensor core truncates it to
                // tf32), A_lo = C - trunc(C) exactly (truncated to tf32 by the
                // tensor core in turn: < 2^-22 |c| per element, < 3e-7 on a
                // unit dot).  The rounding split cost 4 ALU operations per
                // element, and the converters were on the critical path.
                uint32_t hi[32], lo[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint4 v = src[j ^ (lane & 7)];
                    hi[4 * j + 0] = v.x;
                    hi[4 * j + 1] = v.y;
                    hi[4 * j + 2] = v.z;
                    hi[4 * j + 3] = v.w;
                    lo[4 * j + 0] = lo_trunc(v.x);
                    lo[4 * j + 1] = lo_trunc(v.y);
                    lo[4 * j + 2] = lo_trunc(v.z);
                    lo[4 * j + 3] = lo_trunc(v.w);
                }
                if (kc == kChunks - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(raw_empty(s));  // box consumed
                }
                mbar_wait(ops_empty(o), ((go / kOps) & 1) ^ 1);
                if (warp == 4 && lane == 0) trace_stamp(dbg, 2, go);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t col = tmem_base + lane_off + kOpsCol0 + o * 64;
                if (!(dbg & 4)) {  // dbg & 4: no TMEM stores (pipeline experiment)
                    tmem_st32(col, hi);
                    tmem_st32(col + 32, lo);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(ops_full(o));
                if (warp == 4 && lane == 0) trace_stamp(dbg, 3, go);
                if (warp == 7 && lane == 0) trace_stamp(dbg, 7, go);
            }
        }
    } else if (warp >= 8) {
        // ---------------- epilogue: two groups of 4 warps take alternate tiles
        // (group = accumulator); thread = centroid row (lane quarter q)
        const uint32_t q = warp & 3, ew = warp - 8, grp = ew >> 2;
        // lane = query token after the transpose: this warp's best NP
        // (score, centroid) pairs for it, descending.  Centroids arrive in
        // increasing id order, so a later one enters only with a strictly
        // larger score (reference tie order).  thr: the NP-th score (-inf
        // until full); gb: a bound some list in the grid already reached
        // (ties at gb are kept)
        float top_s[QB][NP];
        uint32_t top_i[QB][NP];
        float gb[QB];
#pragma unroll
        for (int qi = 0; qi < QB; ++qi) {
#pragma unroll
            for (int j = 0; j < NP; ++j) top_s[qi][j] = -INFINITY, top_i[qi][j] = 0;
            gb[qi] = -INFINITY;
        }
        const bool tok = lane < rows;
        float* tr = reinterpret_cast<float*>(smem + kOffTr) + ew * 32 * 33;
        uint32_t lt = grp;
        for (uint64_t t = blockIdx.x + uint64_t(grp) * gridDim.x; t < ntiles; t += 2ull * gridDim.x, lt += 2) {
            const uint32_t acc = grp;
            mbar_wait(tfull_bar(acc), (lt >> 1) & 1);
            if (ew == 0 && lane == 0) trace_stamp(dbg, 5, lt);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * kAccCols;
            const uint64_t c0 = t * 128 + q * 32;
            const uint64_t c = c0 + lane;
            const bool valid = c < K;
            // centroids of this lane quarter (0 past the end of a partial last tile)
            const uint32_t nv = c0 >= K ? 0u : (K - c0 < 32 ? uint32_t(K - c0) : 32u);
#pragma unroll
            for (int qi = 0; qi < QB; ++qi) {
                uint32_t rh[32], rl[32];
                tmem_ld32(taddr + 32 * qi, rh);
                tmem_ld32(taddr + 32 * QB + 32 * qi, rl);
                tmem_ld_wait();
                if (qi == QB - 1) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty_bar(acc));
                }
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(__uint_as_float(rh[j]), __uint_as_float(rl[j]));
                float m = -INFINITY;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (uint32_t(j) < rows) m = fmaxf(m, v[j]);
                const uint32_t kw = __ballot_sync(0xffffffffu, valid && m >= t_cs);
                if (lane == 0 && c0 < K) out.keep[qi][c0 >> 5] = kw;
                // 32x32 transpose: tr[centroid][token], pitch 33 (conflict-free both ways)
                __syncwarp();  // the previous query's reads of tr are done
#pragma unroll
                for (int j = 0; j < 32; ++j) tr[lane * 33 + j] = v[j];
                __syncwarp();
                if (tok) {
                    const uint32_t cb = cthr[32 * qi + lane];
                    if (cb) gb[qi] = fmaxf(gb[qi], dev::unord_f32(cb));
                }
                const float thr0 = top_s[qi][NP - 1];
                uint32_t cand = 0;
                float* Sq = out.S[qi];
                // S rows from the transposed tile: one coalesced 128-byte row per
                // centroid (lane = token)
#pragma unroll
                for (int r = 0; r < 32; ++r) {
                    const float sc = tr[r * 33 + lane];
                    cand |= (uint32_t(r) < nv && tok && sc > thr0 && sc >= gb[qi]) ? (1u << r) : 0u;
                    if (uint32_t(r) < nv && !(dbg & 2)) Sq[(c0 + r) * kScoresPitch + lane] = sc;
                }
                // per-lane inserts, rare once the bounds have risen
                while (cand) {
                    const int r = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const float sc = tr[r * 33 + lane];
                    if (sc > top_s[qi][NP - 1] && sc >= gb[qi]) {
                        const uint32_t id = uint32_t(c0 + r);
                        // shift-insert; every position reads only old values
#pragma unroll
                        for (int j = NP - 1; j > 0; --j) {
                            const bool up = sc > top_s[qi][j - 1], here = sc > top_s[qi][j];
                            top_i[qi][j] = up ? top_i[qi][j - 1] : (here ? id : top_i[qi][j]);
                            top_s[qi][j] = up ? top_s[qi][j - 1] : (here ? sc : top_s[qi][j]);
                        }
                        if (sc > top_s[qi][0]) top_s[qi][0] = sc, top_i[qi][0] = id;
                    }
                }
                const float thr = top_s[qi][NP - 1];
                // bounds: CTA-wide in shared memory every tile; one warp trades it
                // with the grid-wide `gthr` every 4th of its tiles (one L2 line
                // that every CTA hits, so per-tile traffic there would serialise)
                if (tok && thr > thr0 && thr > gb[qi]) {
                    atomicMax(const_cast<uint32_t*>(&cthr[32 * qi + lane]), dev::ord_f32(thr));
                    gb[qi] = thr;
                }
                if (ew == kEpiWarps - 1 && (lt & 7) == 7 && tok) {
                    const uint32_t mine = cthr[32 * qi + lane];
                    const uint32_t go = mine ? atomicMax(out.gthr[qi] + lane, mine) : __ldcg(out.gthr[qi] + lane);
                    if (go > mine) atomicMax(const_cast<uint32_t*>(&cthr[32 * qi + lane]), go);
                }
            }
            if (ew == 0 && lane == 0) trace_stamp(dbg, 6, lt);
        }
        if constexpr (NP <= 8) {
            // one list per CTA and token: the 8 epilogue warps' lists merged
            // here (through the transpose buffer, free once every epilogue
            // warp is done), so the consumers merge 148 lists, not 1184
            uint64_t* kx = reinterpret_cast<uint64_t*>(smem + kOffTr);  // [QB][8 warps][32 tokens][NP]
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
#pragma unroll
            for (int qi = 0; qi < QB; ++qi)
#pragma unroll
                for (int j = 0; j < NP; ++j)
                    kx[((qi * kEpiWarps + ew) * 32 + lane) * NP + j] =
                        top_s[qi][j] == -INFINITY ? 0 : dev::make_key(top_s[qi][j], top_i[qi][j]);
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            if (ew < uint32_t(QB)) {
                uint64_t top[NP];
#pragma unroll
                for (int j = 0; j < NP; ++j) top[j] = 0;
                for (uint32_t w = 0; w < kEpiWarps; ++w)
#pragma unroll
                    for (int j = 0; j < NP; ++j) dev::topn_insert<NP>(top, kx[((ew * kEpiWarps + w) * 32 + lane) * NP + j]);
                uint64_t* po = out.partial[ew] + (uint64_t(blockIdx.x) * 32 + lane) * NP;
#pragma unroll
                for (int j = 0; j < NP; ++j) po[j] = top[j];
            }
        } else {
#pragma unroll
            for (int qi = 0; qi < QB; ++qi) {
                uint64_t* po = out.partial[qi] + ((uint64_t(blockIdx.x) * kEpiWarps + ew) * 32 + lane) * NP;
#pragma unroll
                for (int j = 0; j < NP; ++j)
                    po[j] = top_s[qi][j] == -INFINITY ? 0 : dev::make_key(top_s[qi][j], top_i[qi][j]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    cta_stamp(dbg, 1);
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

template <int NP, int QB>
void launch_tf32(const CUtensorMap& map, const IndexView& ix, const TfOut& out, uint32_t rows, float t_cs,
                 uint32_t grid, cudaStream_t st) {
    static launch::PerDeviceOnce configured;
    if (configured.first()) {
        cudaFuncSetAttribute(scores_tf32_kernel<NP, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TfCfg<QB>::kSmemBytes);
    }
    static const uint32_t dbg = [] {
        const char* e = getenv("PLAID_TF32_DBG");
        return e ? uint32_t(atoi(e)) : 0u;
    }();
    ::plaid::launch::pdl(scores_tf32_kernel<NP, QB>, grid, kThreads, TfCfg<QB>::kSmemBytes, st, map, ix.K, out, rows,
                         t_cs, dbg);
    launch::count_launch();
}

template <int QB>
void launch_tf32_np(const CUtensorMap& map, const IndexView& ix, const TfOut& out, uint32_t rows, float t_cs,
                    uint32_t np_bucket, uint32_t grid, cudaStream_t st) {
    switch (np_bucket) {
        case 1: launch_tf32<1, QB>(map, ix, out, rows, t_cs, grid, st); break;
        case 2: launch_tf32<2, QB>(map, ix, out, rows, t_cs, grid, st); break;
        case 4: launch_tf32<4, QB>(map, ix, out, rows, t_cs, grid, st); break;
        case 8: launch_tf32<8, QB>(map, ix, out, rows, t_cs, grid, st); break;
        case 16: if constexpr (QB == 1) { launch_tf32<16, QB>(map, ix, out, rows, t_cs, grid, st); break; }
        [[fallthrough]];
        default:
            if constexpr (QB == 1) launch_tf32<32, QB>(map, ix, out, rows, t_cs, grid, st);
            else launch::fail_cuda_driver(1, "batched S_cq supports nprobe <= 8");
            break;
    }
}

// Test knob (plaid_debug_set_tf32_grid): cap the persistent grid so a small K
// still runs many tiles per CTA (TMA ring wrap, both accumulator groups, the
// grid-wide bound exchange).  0 = one CTA per SM.
std::atomic<uint32_t> g_tf32_grid_cap{0};

uint32_t tf32_grid(const IndexView& ix) {
    const uint64_t ntiles = (ix.K + 127) / 128;
    uint64_t cap = uint64_t(sm_count());
    const uint32_t dbg_cap = g_tf32_grid_cap.load(std::memory_order_relaxed);
    if (dbg_cap && dbg_cap < cap) cap = dbg_cap;
    uint32_t grid = uint32_t(ntiles < cap ? ntiles : cap);
    return grid ? grid : 1;
}

}  // namespace

namespace launch {

bool tensor_scores_supported(const IndexView& ix) { return ix.dim == kDim && ix.K < (1ull << 31); }

void make_centroid_tensor_map(const IndexView& ix, void* out_map) {
    CUtensorMap* map = static_cast<CUtensorMap*>(out_map);
    // 3-D view (32 fp32, centroid, 32-dim chunk): one box = 32 centroids x
    // 4 chunks = 16 KB contiguous in HBM, laid out [chunk][centroid][32] in
    // shared memory (128-B rows, SWIZZLE_128B by centroid & 7)
    const cuuint64_t dims[3] = {32, cuuint64_t(ix.K), cuuint64_t(kDim / 32)};
    const cuuint64_t strides[2] = {cuuint64_t(kDim) * sizeof(float), 32 * sizeof(float)};
    const cuuint32_t box[3] = {32, 32, kDim / 32};
    const cuuint32_t estr[3] = {1, 1, 1};
    // through the runtime's driver entry point: the library does not link
    // libcuda, so it loads (and exports its ABI) on hosts without a driver
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
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ix.centroids), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail_cuda_driver(int(r), "cuTensorMapEncodeTiled");
}

uint32_t scores_tensor_max_warps() { return uint32_t(sm_count()) * kEpiWarps; }

uint32_t scores_tensor(const void* cmap, const IndexView& ix, const float* d_q, uint32_t rows, float t_cs,
                       float* d_scores, uint32_t* d_keep_bits, uint64_t* d_partial, uint32_t np_bucket,
                       uint32_t* d_gthr, cudaStream_t st) {
    const CUtensorMap& map = *static_cast<const CUtensorMap*>(cmap);
    TfOut out{};
    out.Q[0] = d_q, out.S[0] = d_scores, out.keep[0] = d_keep_bits, out.partial[0] = d_partial, out.gthr[0] = d_gthr;
    const uint32_t grid = tf32_grid(ix);
    launch_tf32_np<1>(map, ix, out, rows, t_cs, np_bucket, grid, st);
    return np_bucket <= 8 ? grid : grid * kEpiWarps;  // one list per CTA (merged in the epilogue) up to NP = 8
}

uint32_t scores_tensor_batch(const void* cmap, const IndexView& ix, const TfOut& out, uint32_t qb, uint32_t rows,
                             float t_cs, uint32_t np_bucket, cudaStream_t st) {
    const CUtensorMap& map = *static_cast<const CUtensorMap*>(cmap);
    const uint32_t grid = tf32_grid(ix);
    if (qb == 1) launch_tf32_np<1>(map, ix, out, rows, t_cs, np_bucket, grid, st);
    else launch_tf32_np<2>(map, ix, out, rows, t_cs, np_bucket, grid, st);
    return np_bucket <= 8 ? grid : grid * kEpiWarps;
}

}  // namespace launch
}  // namespace plaid

// Debug: copy the pipeline timeline (see trace_stamp / cta_stamp) to the host:
// out[0..2048) = CTA 0 events, out[2048..2560) = per-CTA begin/end.
// Test knob: cap the S_cq grid at `ctas` CTAs (0 = one per SM); returns the old cap.
extern "C" uint32_t plaid_debug_set_tf32_grid(uint32_t ctas) { return plaid::g_tf32_grid_cap.exchange(ctas); }

extern "C" int plaid_debug_tf32_trace(unsigned long long* out) {
    int rc = int(cudaMemcpyFromSymbol(out, plaid::g_tf32_trace, sizeof(plaid::g_tf32_trace)));
    if (!rc) rc = int(cudaMemcpyFromSymbol(out + 8 * 256, plaid::g_tf32_cta, sizeof(plaid::g_tf32_cta)));
    return rc;
}
