// Dependent-chain latencies of the warp-wide primitives the pivot searches are built from
// (one warp, one SM): cycles per op = (clock64 around N dependent ops) / N.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/warp_lat tools/micro/warp_lat.cu
#include <cstdint>
#include <cstdio>
#define FULL 0xffffffffu
constexpr int N = 4096;

template <int MODE>
__global__ void k(uint32_t seed, long long* out, uint32_t* sink) {
    const int lane = threadIdx.x & 31;
    uint32_t x = seed + lane, y = seed * 3 + lane;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if (MODE == 0) x = x * 3 + 1;                                      // IMAD chain
        if (MODE == 1) x = __reduce_min_sync(FULL, x ^ lane) + 1;          // redux.min -> ALU
        if (MODE == 2) x = __ballot_sync(FULL, (x >> lane) & 1) + 1;       // vote.ballot -> ALU
        if (MODE == 3) x = __shfl_sync(FULL, x, x & 31) + 1;               // shfl.idx (data-dependent lane)
        if (MODE == 4) {                                                    // redux -> shfl (the row-form step)
            const uint32_t m = __reduce_min_sync(FULL, x ^ lane);
            x = __shfl_sync(FULL, y, m & 31) + m;
        }
        if (MODE == 5) {                                                    // ballot -> ffs -> shfl
            const uint32_t b = __ballot_sync(FULL, (x >> lane) & 1) | 0x80000000u;
            x = __shfl_sync(FULL, y, __ffs(b) - 1) + b;
        }
        if (MODE == 6) x = __match_any_sync(FULL, x & 3) + 1;              // match.any
        if (MODE == 7) x = (x & (0u - x)) + 3;                              // x & -x chain (2 ALU)
        if (MODE == 8) {                                                    // shfl.idx, fixed lane pattern
            x = __shfl_sync(FULL, x, i & 31) + 1;
        }
        if (MODE == 9) {                                                    // 128-bit neg carry chain + and
            unsigned long long lo = x, hi = y, nlo, nhi;
            asm("sub.cc.u64 %0, 0, %2;\n\tsubc.u64 %1, 0, %3;\n" : "=l"(nlo), "=l"(nhi) : "l"(lo), "l"(hi));
            x = (uint32_t)(nlo & lo) + 5; y = (uint32_t)(nhi & hi) + 1;
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[MODE] = t1 - t0;
    sink[threadIdx.x] = x + y;
}

int main() {
    long long* out; uint32_t* sink;
    cudaMallocManaged(&out, 16 * sizeof(long long));
    cudaMalloc(&sink, 1024 * 4);
    const char* nm[] = {"imad", "redux.min+add", "ballot+add", "shfl.idx(dep lane)+add", "redux->shfl", "ballot->ffs->shfl",
                        "match.any+add", "x&-x +add (3 ALU)", "shfl.idx(fixed lane)+add", "neg128+and+add"};
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32>>>(rep + 1, out, sink); k<1><<<1, 32>>>(rep + 1, out, sink); k<2><<<1, 32>>>(rep + 1, out, sink);
        k<3><<<1, 32>>>(rep + 1, out, sink); k<4><<<1, 32>>>(rep + 1, out, sink); k<5><<<1, 32>>>(rep + 1, out, sink);
        k<6><<<1, 32>>>(rep + 1, out, sink); k<7><<<1, 32>>>(rep + 1, out, sink); k<8><<<1, 32>>>(rep + 1, out, sink);
        k<9><<<1, 32>>>(rep + 1, out, sink);
        cudaDeviceSynchronize();
    }
    for (int m = 0; m < 10; ++m) printf("%-28s %6.1f cycles per iteration\n", nm[m], (double)out[m] / N);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
