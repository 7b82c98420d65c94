// Throughput of VOTE (ballot), SHFL and a smem-based bit transpose, 32 warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(long long* out, uint64_t seed, int iters) {
    __shared__ uint32_t sm[1024 * 2];
    uint64_t w = seed * (threadIdx.x + 1) * 0x9e3779b97f4a7c15ull;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= __ballot_sync(0xffffffffu, (w >> j) & 1ull);
        } else if (MODE == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= __shfl_sync(0xffffffffu, static_cast<uint32_t>(w) + j, j);
        } else if (MODE == 2) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(w) + acc, j & 31);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += __popc(static_cast<uint32_t>(w >> j) ^ acc);
        }
        w = w * 6364136223846793005ull + 1442695040888963407ull;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 0x12345) out[1] = acc;
}

template <int MODE>
void run(const char* name, int nthreads) {
    long long* d;
    cudaMalloc(&d, 16);
    const int iters = 100;
    k<MODE><<<1, nthreads>>>(d, 7, iters);
    k<MODE><<<1, nthreads>>>(d, 7, iters);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double ops = 32.0 * iters * (nthreads / 32);
    printf("%-12s threads=%4d: %lld cycles, %.2f cycles per warp-op (SM-wide)\n", name, nthreads, h[0], h[0] / ops);
}

int main() {
    for (int nt : {32, 128, 1024}) {
        run<0>("ballot", nt);
        run<1>("shfl.idx", nt);
        run<2>("shfl.xor dep", nt);
        run<3>("alu", nt);
    }
}
