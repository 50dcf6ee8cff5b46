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

template <int N, bool TS>
__global__ void bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 128 * 128 + N * 128; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 128 * 4);
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tm + (it & 1) * 256;  // two accumulators (<= 256 cols each)
            if (TS) {
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
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N, bool TS>
void run(unsigned long long* d, int iters) {
    const int smem = 128 * 128 * 4 + 256 * 128 * 4 + 2048;
    cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<N, TS><<<1, 128, smem>>>(d, iters);
    cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d %s: %.1f cycles/MMA (%s)\n", N, TS ? "TS" : "SS", double(h) / iters,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 148);
    const int it = 4096;
    run<32, false>(d, it);
    run<32, true>(d, it);
    run<64, false>(d, it);
    run<128, false>(d, it);
    run<256, false>(d, it);
    run<256, true>(d, it);
    return 0;
}
