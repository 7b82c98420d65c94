// Achievable SMEM lookup rate: 16 warps, each quarter-warp reads one random 128-B table
// row per LDS.128 (the M4RM lookup pattern), with and without a table-build stream.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k(long long* out, int iters) {
    extern __shared__ __align__(128) uint64_t T[];  // 256 x 16 words (32 KB) x 2
    const int tid = threadIdx.x, lane = tid & 31, wp = lane & 7;
    for (int i = tid; i < 2 * 256 * 16; i += NW * 32) T[i] = i * 0x9e3779b97f4a7c15ull;
    __syncthreads();
    uint32_t idx = tid * 2654435761u;
    uint64_t a0 = 0, a1 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            idx = idx * 1664525u + 1013904223u;
            const uint64_t* e = T + ((idx >> 24) & 255) * 16 + 2 * wp;
            uint4 v;
            const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(e));
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
            a0 ^= v.x | ((uint64_t)v.y << 32);
            a1 ^= v.z | ((uint64_t)v.w << 32);
        }
        if (MODE == 1) __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
    if ((a0 ^ a1) == 0x123) out[1] = a0;
}

template <int NW, int MODE>
void run(const char* name) {
    long long* d;
    cudaMalloc(&d, 16);
    const size_t sm = 2 * 256 * 16 * 8;
    cudaFuncSetAttribute(k<NW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int iters = 1000;
    k<NW, MODE><<<1, NW * 32, sm>>>(d, iters);
    k<NW, MODE><<<1, NW * 32, sm>>>(d, iters);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double wavefronts = (double)iters * 16 * NW * 4;  // 4 wavefronts per LDS.128 (4 rows x 128 B)
    printf("%-22s warps=%2d: %.3f wavefronts/clk\n", name, NW, wavefronts / h[0]);
}

int main() {
    run<8, 0>("lookups");
    run<16, 0>("lookups");
    run<32, 0>("lookups");
    run<16, 1>("lookups+syncthreads");
}
