// Cycles per pivot step of the warp-level leaf search, with parts removed.
#include <cstdio>
#include <cstdint>
#define FULL 0xffffffffu
__device__ __forceinline__ uint64_t above(int c) { return c >= 63 ? 0ull : (~0ull << (c + 1)); }

__global__ void k3(const uint64_t* rows, long long* out, long long* P, int* Q) {
    __shared__ uint64_t s_u[64], s_uf[64];
    __shared__ int s_q[64];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    uint64_t w = rows[lane];
    int src = lane;
    int p = 0, col = 0, t = 0;
    long long t0 = clock64();
#pragma unroll 1
    while (col < 64 && p < 32) {
        const int pr = p;
        // speculative, independent of the ballot
        const uint64_t wp = __shfl_sync(FULL, w, pr);
        const int psrc = __shfl_sync(FULL, src, pr);
        const uint32_t wl32 = col < 32 ? (uint32_t)w : (uint32_t)(w >> 32);
        const unsigned hit = __ballot_sync(FULL, lane >= pr && ((wl32 >> (col & 31)) & 1u));
        if (hit == 0) { col++; continue; }
        const int ln = __ffs(hit) - 1;
        const uint64_t u = __shfl_sync(FULL, w, ln);
        const int usrc = __shfl_sync(FULL, src, ln);
        const uint64_t am = above(col);
        w = lane == ln ? wp : w;
        src = lane == ln ? psrc : src;
        w = lane == pr ? u : w;
        src = lane == pr ? usrc : src;
        const uint64_t us = u & am;
        const bool e = lane > pr && ((w >> col) & 1ull);
        w ^= e ? us : 0ull;
        if (lane == 0) {
            s_u[t] = us; s_uf[t] = u; s_q[t] = col;
            P[p] = ln; Q[p] = col;
        }
        ++t; ++p; ++col;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = (t1 - t0); out[1] = t; out[2] = s_u[0] ^ s_uf[1] ^ s_q[2] ^ src; }
}

template <int V>
__global__ void k(const uint64_t* rows, long long* out, long long* P, int* Q) {
    __shared__ uint64_t s_u[64], s_uf[64];
    __shared__ int s_q[64];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    uint64_t w = rows[lane];
    int src = lane;
    int p = 0, col = 0, t = 0;
    long long t0 = clock64();
    while (col < 64 && p < 32) {
        const int pr = p;
        const bool cand = lane >= pr;
        unsigned hit = __ballot_sync(FULL, cand && ((w >> col) & 1ull));
        int cstar = col;
        if (hit == 0) { col++; continue; }
        const int ln = __ffs(hit) - 1;
        const uint64_t u = __shfl_sync(FULL, w, ln);
        if (V != 2 && ln != pr) {
            const uint64_t wp = __shfl_sync(FULL, w, pr);
            const int usrc = __shfl_sync(FULL, src, ln);
            const int psrc = __shfl_sync(FULL, src, pr);
            if (lane == ln) { w = wp; src = psrc; }
            if (lane == pr) { w = u; src = usrc; }
        }
        const uint64_t us = u & above(cstar);
        if (lane > pr && ((w >> cstar) & 1ull)) w ^= us;
        if (V == 0 && lane == 0) {
            s_u[t] = us; s_uf[t] = u; s_q[t] = cstar;
            P[p] = ln; Q[p] = cstar;
        }
        ++t; ++p; col = cstar + 1;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = (t1 - t0); out[1] = t; out[2] = s_u[0] ^ s_uf[1] ^ s_q[2] ^ src; }
}
int main() {
    uint64_t h[32];
    uint64_t s = 12345;
    for (int i = 0; i < 32; ++i) { s = s * 6364136223846793005ull + 1442695040888963407ull; h[i] = s ^ (s >> 29); }
    uint64_t* d; long long *o, *P; int* Q;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 64); cudaMalloc(&P, 8 * 64); cudaMalloc(&Q, 4 * 64);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    long long r[3];
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 1024>>>(d, o, P, Q); cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost); if (rep) printf("full      : %lld cycles / %lld pivots = %lld\n", r[0], r[1], r[0] / r[1]);
        k<1><<<1, 1024>>>(d, o, P, Q); cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost); if (rep) printf("no stores : %lld cycles / %lld pivots = %lld\n", r[0], r[1], r[0] / r[1]);
        k<2><<<1, 1024>>>(d, o, P, Q); cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost); if (rep) printf("no swap   : %lld cycles / %lld pivots = %lld\n", r[0], r[1], r[0] / r[1]);
        k<0><<<1, 32>>>(d, o, P, Q); cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost); if (rep) printf("full,32thr: %lld cycles / %lld pivots = %lld\n", r[0], r[1], r[0] / r[1]);
        k3<<<1, 32>>>(d, o, P, Q); cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost); if (rep) printf("branchless: %lld cycles / %lld pivots = %lld\n", r[0], r[1], r[0] / r[1]);
    }
}
