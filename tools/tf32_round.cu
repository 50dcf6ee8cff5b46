// tf32_round.cu — does tcgen05.mma.kind::tf32 truncate or round the low 13
// mantissa bits of fp32 operands?  A = 1 + 0.75*2^-10 everywhere, B = 1.0:
// D[0][0] = 8 * tf32(A) = 8.0 (truncate) or 8.0078125 (round to nearest).
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

__global__ void k(float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    float* a = reinterpret_cast<float*>(sm);
    float* b = reinterpret_cast<float*>(sm + 128 * 32 * 4);
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) a[i] = 1.0f + 0.75f * 0.0009765625f;
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) b[i] = 1.0f;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    if (threadIdx.x == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(desc(smem_u32(a))), "l"(desc(smem_u32(b))), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32) {
        uint32_t r;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (threadIdx.x == 0) out[0] = __uint_as_float(r);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(32));
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<1, 128, 64 * 1024>>>(d);
    float h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("D[0][0] = %.9f -> %s (%s)\n", h, h == 8.0f ? "TRUNCATE" : (h == 8.0078125f ? "ROUND" : "?"),
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
