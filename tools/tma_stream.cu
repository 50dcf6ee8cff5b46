// tma_stream.cu — how fast can 148 CTAs stream a 128 MiB buffer into shared
// memory with bulk async copies?  The streaming floor of the S_cq kernel
// (which reads C = 2^18 x 128 fp32 once per query).
//   mode 0: 1-D cp.async.bulk of 16 KB contiguous chunks
//   mode 1: plain LDG.128 by all threads (no smem), for comparison
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int SLOTS>
__global__ void __launch_bounds__(128, 1) bulk_stream(const uint8_t* src, uint64_t chunks, uint64_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[SLOTS];
    const uint32_t chunk_bytes = 16384;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SLOTS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint64_t acc = 0;
    if (threadIdx.x == 0) {
        uint64_t issued = 0, done = 0;
        const uint64_t mine = (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
        auto issue = [&](uint64_t i) {
            const int s = int(i % SLOTS);
            const uint64_t c = blockIdx.x + i * gridDim.x;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(chunk_bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(sm + s * chunk_bytes)),
                         "l"(src + c * chunk_bytes), "r"(chunk_bytes), "r"(smem_u32(&full[s]))
                         : "memory");
        };
        for (; issued < mine && issued < SLOTS; ++issued) issue(issued);
        for (; done < mine; ++done) {
            const int s = int(done % SLOTS);
            const uint32_t par = uint32_t(done / SLOTS) & 1;
            asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
                             smem_u32(&full[s])), "r"(par) : "memory");
            acc += sm[s * chunk_bytes];
            if (issued < mine) issue(issued++);
        }
    }
    if (threadIdx.x == 0 && acc == 12345) sink[0] = acc;
}

__global__ void ldg_stream(const uint4* src, uint64_t n16, uint64_t* sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(src + i);
        acc += v.x ^ v.w;
    }
    if (acc == 12345) sink[0] = acc;
}

int main() {
    const uint64_t bytes = 128ull << 20;
    uint8_t* src;
    uint64_t* sink;
    uint8_t* flush;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 8);
    cudaMalloc(&flush, 256ull << 20);
    cudaMemset(src, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 8; ++it) {
            cudaMemset(flush, it, 256ull << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        printf("%-28s %7.1f us  %6.0f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    const uint64_t chunks = bytes / 16384;
    cudaFuncSetAttribute(bulk_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
    cudaFuncSetAttribute(bulk_stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    cudaFuncSetAttribute(bulk_stream<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384);
    run("bulk 16KB x4 slots, 148 CTAs", [&] { bulk_stream<4><<<148, 128, 4 * 16384>>>(src, chunks, sink); });
    run("bulk 16KB x8 slots, 148 CTAs", [&] { bulk_stream<8><<<148, 128, 8 * 16384>>>(src, chunks, sink); });
    run("bulk 16KB x13 slots, 148 CTAs", [&] { bulk_stream<13><<<148, 128, 13 * 16384>>>(src, chunks, sink); });
    run("ldg.128, 148x8 CTAs x 256", [&] { ldg_stream<<<148 * 8, 256>>>((const uint4*)src, bytes / 16, sink); });
    run("ldg.128, 148x32 CTAs x 256", [&] { ldg_stream<<<148 * 32, 256>>>((const uint4*)src, bytes / 16, sink); });
    return 0;
}
