// mma_bench.cu — microbenchmark: cycles per tcgen05.mma.kind::tf32 (M=128,
// K=8) as a function of N and of A's source (smem "SS" vs TMEM "TS").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench mma_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    uint64_t d = uint64_t((addr >> 4) & 0x3FFFu);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

template <int N, bool TS, int CONT = 0, int NACC = 2, int MIX = 0, int CE = 0>
__global__ void bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, bar2;
    const uint32_t warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 128 * 128 + N * 128; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 128 * 4);
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (CONT && warp >= 1 && warp < 1 + CONT) {
        // TMEM traffic on columns [384, 448) of this warp's lane quarter
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = j;
        const uint32_t ta = tm + ((warp & 3) * 32 << 16) + 384;
        while (!stop) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),
                "r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = NACC == 1 ? tm : NACC == 2 ? tm + (it & 1) * 256 : tm + (it & 3) * 64;
            if (MIX) {
                // the S_cq pattern: C_hi . [Q_hi | Q_lo] (N) then C_lo . Q_hi (N/2 when MIX = 1) into one D
                const uint32_t idesc2 = MIX == 1 ? ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(N / 2) >> 3) << 17) |
                                                    ((128u >> 4) << 24))
                                                 : idesc;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tm + 256 + 8 * (it & 3)), "l"(desc(b + (it & 3) * 32)), "r"(idesc), "r"(it > 1 ? 1 : 0));
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tm + 288 + 8 * (it & 3)), "l"(desc(b + (it & 3) * 32)), "r"(idesc2), "r"(1));
                if (CE && (it % CE) == CE - 1)  // a commit every CE iterations (the S_cq loop commits per chunk)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&bar2)));
            } else if (TS) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tm + 256 + 32 * 0), "l"(desc(b + (it & 3) * 32)), "r"(idesc), "r"(it > 1 ? 1 : 0));
            } else {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(desc(a + (it & 3) * 32)), "l"(desc(b + (it & 3) * 32)), "r"(idesc), "r"(it > 1 ? 1 : 0));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        stop = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N, bool TS, int CONT = 0, int NACC = 2, int MIX = 0, int CE = 0>
void run(unsigned long long* d, int iters) {
    const int smem = 128 * 128 * 4 + 256 * 128 * 4 + 2048;
    cudaFuncSetAttribute(bench<N, TS, CONT, NACC, MIX, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<N, TS, CONT, NACC, MIX, CE><<<1, 128, smem>>>(d, iters);
    cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d %s cont=%d nacc=%d mix=%d commit/%d: %.1f cycles/MMA (%s)\n", N, TS ? "TS" : "SS", CONT, NACC, MIX, CE,
           double(h) / iters / (MIX ? 2 : 1),
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 148);
    const int it = 4096;
    run<32, false>(d, it);
    run<32, true>(d, it);
    run<64, false>(d, it);
    run<64, true>(d, it);
    run<96, false>(d, it);
    run<96, true>(d, it);
    run<128, false>(d, it);
    run<128, true>(d, it);
    run<256, false>(d, it);
    run<256, true>(d, it);
    run<64, true, 1>(d, it);
    run<64, true, 3>(d, it);
    run<32, true, 3>(d, it);
    run<64, false, 3>(d, it);
    run<64, true, 0, 1>(d, it);
    run<32, true, 0, 1>(d, it);
    run<64, true, 0, 4>(d, it);
    run<32, true, 0, 4>(d, it);
    run<128, true, 0, 1>(d, it);
    run<64, true, 3, 1>(d, it);
    // the S_cq issue pattern (two MMAs per K step into one accumulator)
    run<64, true, 0, 1, 1>(d, it);
    run<64, true, 0, 1, 2>(d, it);
    run<128, true, 0, 1, 1>(d, it);
    run<128, true, 0, 1, 2>(d, it);
    run<64, true, 3, 1, 1>(d, it);
    run<64, true, 3, 1, 2>(d, it);
    run<64, true, 0, 1, 1, 4>(d, it);
    run<64, true, 0, 1, 1, 1>(d, it);
    return 0;
}
