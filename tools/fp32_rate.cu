// fp32_rate.cu — issue/pipe rate of FMUL2, FADD2(.FTZ), scalar FADD/FMUL on
// sm_100a: cycles per warp-instruction per SMSP with W warps per SMSP.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_rate fp32_rate.cu
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 add2f(u64 a, u64 b) { u64 r; asm volatile("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float addf(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
template <int OP>
__global__ void k(u64* out, int iters, u64 seed) {
    u64 a[8], b = seed | 0x3f8000003f800000ull;
    float f[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + i, f[i] = float(i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = mul2(a[i], b);
            if (OP == 1) a[i] = add2f(a[i], b);
            if (OP == 2) f[i] = addf(f[i], 1.0f);
            if (OP == 3) { a[i] = mul2(a[i], b); f[i] = addf(f[i], 1.0f); }
        }
    }
    long long t1 = clock64();
    u64 s = 0; for (int i = 0; i < 8; ++i) s += a[i] + u64(f[i]);
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (s == 42) out[1] = s;
}
template <int OP> void run(u64* d, int warps_per_smsp) {
    const int it = 4096;
    k<OP><<<1, 128 * warps_per_smsp>>>(d, it, 3);
    cudaDeviceSynchronize();
    u64 h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double instr = double(it) * 8 * warps_per_smsp * (OP == 3 ? 2 : 1);
    printf("op=%d warps/smsp=%d: %.2f cycles per warp-instr per SMSP\n", OP, warps_per_smsp, double(h) / instr);
}
int main() {
    u64* d; cudaMalloc(&d, 16);
    for (int w : {1, 2, 4}) { run<0>(d, w); run<1>(d, w); run<2>(d, w); run<3>(d, w); }
    return 0;
}
