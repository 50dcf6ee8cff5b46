// pdl_chain.cu — the fixed cost of one kernel boundary in a dependent chain:
// N tiny kernels (each reads a word the previous one wrote, writes one), with
// and without programmatic dependent launch, timed with events.  The
// 17-kernel PLAID query pays this N times.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_chain pdl_chain.cu
#include <cstdint>
#include <cstdio>

__global__ void step(const uint32_t* in, uint32_t* out, int grid_wide) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t v = *reinterpret_cast<const volatile uint32_t*>(in);
    if (grid_wide || (blockIdx.x == 0 && threadIdx.x == 0)) out[blockIdx.x * blockDim.x + threadIdx.x] = v + 1;
}

int main() {
    uint32_t* buf;
    cudaMalloc(&buf, 64 << 20);
    cudaMemset(buf, 0, 64 << 20);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int pdl = 0; pdl < 2; ++pdl)
        for (int grid : {1, 148, 1184}) {
            const int n = 32;
            float best = 1e9;
            for (int it = 0; it < 20; ++it) {
                cudaEventRecord(a, st);
                for (int i = 0; i < n; ++i) {
                    cudaLaunchConfig_t cfg{};
                    cfg.gridDim = grid;
                    cfg.blockDim = 256;
                    cfg.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = pdl;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    uint32_t* in = buf + (i % 2) * (8 << 20);
                    uint32_t* out = buf + ((i + 1) % 2) * (8 << 20);
                    cudaLaunchKernelEx(&cfg, step, (const uint32_t*)in, out, 1);
                }
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (it > 2 && ms < best) best = ms;
            }
            printf("pdl=%d grid=%4d: %.2f us per dependent kernel (%s)\n", pdl, grid, best * 1e3 / n,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
