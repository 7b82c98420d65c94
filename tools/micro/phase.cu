// Microbenchmark: cost of one "solve group" step (table build by Gray segments +
// X update + 2 __syncthreads) in a CTA of NT threads, all data in shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kW = 16;
struct Info { uint64_t uf[64]; int q[64]; int pos[64]; int gs[9]; uint8_t rb[64]; int kb; };

template <int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) k(long long* out, int reps) {
    extern __shared__ uint64_t sm[];
    __shared__ Info L;
    uint64_t* X = sm;            // 64 x 16
    uint64_t* tb = sm + 64 * kW; // 256 x 16
    const int tid = threadIdx.x;
    if (tid < 64) { L.uf[tid] = 0x9e3779b97f4a7c15ull * (tid + 1); L.q[tid] = tid; L.pos[tid] = tid; L.rb[tid] = tid * 37; }
    if (tid < 9) L.gs[tid] = 8 * tid;
    if (tid == 0) L.kb = 64;
    for (int i = tid; i < 64 * kW; i += NT) X[i] = i * 0x1234567ull;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep)
    for (int g = 0; g < 8; ++g) {
        const int g0 = L.gs[g], g1 = L.gs[g + 1];
        if (MODE != 2) {
        for (int base = 0; base < 1024; base += NT) {
            const int t2 = base + tid;
            const int seg = t2 >> 7, el = (t2 >> 3) & 15, tw = t2 & 7;
            uint64_t v0[8], v1[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int r = L.pos[8 * g + b];
                v0[b] = r >= 0 ? X[r * kW + 2 * tw] : 0ull;
                v1[b] = r >= 0 ? X[r * kW + 2 * tw + 1] : 0ull;
            }
            uint64_t l0 = 0, l1 = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) if ((el >> b) & 1) { l0 ^= v0[b]; l1 ^= v1[b]; }
            const int kk = 2 * seg, eh0 = kk ^ (kk >> 1), eh1 = (kk + 1) ^ ((kk + 1) >> 1);
#pragma unroll
            for (int b = 0; b < 4; ++b) if ((eh0 >> b) & 1) { l0 ^= v0[4 + b]; l1 ^= v1[4 + b]; }
            uint64_t* e = tb + (eh0 * 16 + el) * kW + 2 * tw;
            e[0] = l0; e[1] = l1;
            e = tb + (eh1 * 16 + el) * kW + 2 * tw;
            e[0] = l0 ^ v0[4]; e[1] = l1 ^ v1[4];
        }
        }
        if (MODE != 1) __syncthreads();
        if (MODE != 2) {
        for (int i = tid; i < (64 - g0) * kW; i += NT) {
            const int t = g0 + i / kW, kq = i % kW;
            unsigned cb = static_cast<unsigned>(L.uf[t] >> (8 * g)) & 0xffu;
            if (t < g1) cb &= (1u << (L.q[t] - 8 * g)) - 1u;
            unsigned m = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) if ((cb >> b) & 1u) m ^= L.rb[8 * g + b];
            X[t * kW + kq] ^= tb[m * kW + kq];
        }
        }
        if (MODE != 1) __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / reps;
    if (tid == 1) out[1] = X[5];
}

template <int NT, int MODE>
void run(const char* name) {
    long long* d; cudaMalloc(&d, 16);
    size_t sm = sizeof(uint64_t) * (64 * kW + 256 * kW);
    cudaFuncSetAttribute(k<NT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<NT, MODE><<<1, NT, sm>>>(d, 10);
    k<NT, MODE><<<1, NT, sm>>>(d, 10);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s NT=%4d  %lld cycles per 8 groups (%lld per group)  err=%s\n", name, NT, h[0], h[0] / 8,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<1024, 0>("full step");
    run<512, 0>("full step");
    run<256, 0>("full step");
    run<1024, 1>("no syncs");
    run<1024, 2>("syncs only");
    run<256, 2>("syncs only");
}
