// Microbenchmark: throughput of legacy warp-level mma.sync shapes on this GPU.
// Used to decide whether a b1 (AND+POPC) or s8 tensor-core mapping of the GF(2)
// multiply can beat the SMEM-bound M4RM path (SURVEY.md §7 "Hard parts" 8).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k(int iters, int* out) {
    unsigned a0 = threadIdx.x * 0x9e3779b9u, a1 = a0 ^ 0x1234567u, a2 = a0 + 7, a3 = a0 * 3;
    unsigned b0 = a0 ^ 0xdeadbeefu, b1 = a1 + 11;
    int c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (KIND == 0) {
                asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            } else if (KIND == 1) {
                asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            }
        }
    }
    int s = 0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    if (s == 0x7fffffff) out[0] = s;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    const char* names[3] = {"b1 m16n8k256 and.popc", "s8 m16n8k32", "f16 m16n8k16 f32acc"};
    const double kdim[3] = {256, 32, 16};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 128, iters = 4096;
    for (int kind = 0; kind < 3; ++kind) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) k<0><<<blocks, threads>>>(iters, out);
            if (kind == 1) k<1><<<blocks, threads>>>(iters, out);
            if (kind == 2) k<2><<<blocks, threads>>>(iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            double mmas = double(blocks) * (threads / 32) * iters * 8;
            double ops = mmas * 16 * 8 * kdim[kind] * 2;
            if (rep) printf("%-24s %8.3f ms  %10.1f T(bit)op/s  err=%s\n", names[kind], ms, ops / ms / 1e9,
                            cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
