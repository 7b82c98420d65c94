// Dependent-chain latencies of warp collectives on this GPU (cycles per op).
#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, unsigned seed) {
    unsigned v = threadIdx.x * seed + 1;
    long long t0, t1;
    const int N = 1024;
    // SHFL.IDX chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, v & 31) + 1;
    t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / N;
    // REDUX.OR chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __reduce_or_sync(0xffffffffu, v) + threadIdx.x;
    t1 = clock64();
    if (threadIdx.x == 0) out[1] = (t1 - t0) / N;
    // VOTE (ballot) chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __ballot_sync(0xffffffffu, (v >> (threadIdx.x & 31)) & 1) + threadIdx.x;
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = (t1 - t0) / N;
    // LOP3/IADD chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = (v ^ (v >> 3)) + 0x9e3779b9u;
    t1 = clock64();
    if (threadIdx.x == 0) out[3] = (t1 - t0) / N;
    // 64-bit shuffle chain
    unsigned long long w = v;
    t0 = clock64();
    for (int i = 0; i < N; ++i) w = __shfl_sync(0xffffffffu, w, (unsigned)w & 31) + 1;
    t1 = clock64();
    if (threadIdx.x == 0) out[4] = (t1 - t0) / N;
    // __syncwarp chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) { __syncwarp(); v += 1; }
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = (t1 - t0) / N;
    // LDS dependent chain
    __shared__ unsigned sm[64];
    sm[threadIdx.x & 63] = threadIdx.x;
    __syncwarp();
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = sm[(v + i) & 63];
    t1 = clock64();
    if (threadIdx.x == 0) out[6] = (t1 - t0) / N;
    if (v == 0x12345) out[7] = v + w;
}
int main() {
    long long* d; cudaMalloc(&d, 64);
    long long h[8];
    k<<<1, 32>>>(d, 3); cudaDeviceSynchronize();
    k<<<1, 32>>>(d, 3); cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("shfl32 %lld  redux %lld  ballot %lld  alu %lld  shfl64 %lld  syncwarp %lld  lds %lld\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
}
