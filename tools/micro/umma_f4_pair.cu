// The fp4 MMA ceiling of the Schur kernel's data path, 1-SM vs CTA-pair (cta_group::2).
//
// Same operands as the Schur kernel (csrc/schur_f4.cu): E2M1 nibbles, K-major canonical
// no-swizzle layout in 256-element K stages (8-row x 16-byte core matrices, LBO 128 B,
// SBO 1024 B), UE8M0 block-32 scales all 2^0 in TMEM.  Unlike tools/micro/umma_f4.cu the
// issuing thread never drains the pipe: it issues `iters` x 16 MMAs into alternating
// accumulators and commits once, so the figure is the tensor pipe's own rate.
//   peak1: one CTA per SM, M = 128, N = 224 (the Schur kernel's tile)
//   peak2: CTA pairs (cluster of 2), M = 256 (128 A rows per CTA), N = 224, each CTA
//          holding half of B (112 rows) -- per SM, half the B operand reads
// A pair correctness check first: C = A * B^T (256 x 224, K = 1024) from one pair,
// parity of the fp32 counts against the CPU, which also pins which CTA holds which
// half of B.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/umma_f4_pair tools/micro/umma_f4_pair.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("%s: %s\n", #x, cudaGetErrorString(e));                     \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

constexpr int KS = 256, KSB = KS / 2, NST = 4;  // K stage: 256 elements = 128 B per row; K = 1024
constexpr int N_ = 224;
constexpr uint32_t SF = 448;                    // scale-factor columns 448..511 (all 0x7F)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return (uint64_t((addr >> 4) & 0x3FFF)) | (uint64_t(128 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46);
}
template <int M>
__host__ __device__ constexpr uint32_t idesc() {
    return (1u << 7) | (1u << 10) | (1u << 23) | (uint32_t(N_ >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void wait_parity(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(
            su32(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void fill_scales(uint32_t tbase, int warp) {
    if (warp < 4) {
        const uint32_t v = 0x7F7F7F7Fu;
        for (int c = 0; c < 64; c += 8) {
            const uint32_t ta = tbase + (uint32_t(warp * 32) << 16) + SF + c;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta), "r"(v), "r"(v),
                         "r"(v), "r"(v), "r"(v), "r"(v), "r"(v), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
}
// operand row r (of `rows`), K stage s, 16-byte chunk kc -> smem offset (the Schur kernel's layout)
__device__ __forceinline__ int op_off(int r, int s, int kc, int rows) { return s * rows * KSB + (r >> 3) * 1024 + kc * 128 + (r & 7) * 16; }

// fill: A rows then B rows of this CTA from global nibble rows (K/2 bytes each)
__device__ void load_ops(uint8_t* sm, const uint8_t* A8, const uint8_t* B8, int arows, int brows) {
    for (int i = threadIdx.x; i < (arows + brows) * NST * 8; i += blockDim.x) {
        const int row = i / (NST * 8), s = (i / 8) % NST, kc = i % 8;
        const bool isa = row < arows;
        const int r = isa ? row : row - arows;
        const uint8_t* src = (isa ? A8 : B8) + size_t(r) * 512 + s * KSB + kc * 16;
        uint8_t* dst = sm + (isa ? 0 : arows * 512) + op_off(r, s, kc, isa ? arows : brows);
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    }
}

template <int M>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc, uint32_t tsf) {
    if (M == 128)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc<M>()), "r"(acc), "r"(tsf), "r"(tsf + 32));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc<M>()), "r"(acc), "r"(tsf), "r"(tsf + 32));
}

// 16 MMAs = K 1024 (4 stages x 4 K-steps) into accumulator `acc`
template <int M>
__device__ __forceinline__ void issue_k(uint32_t tbase, uint32_t acc, uint32_t a, uint32_t b, int brows) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int s = j >> 2, k = j & 3;
        mma<M>(tbase + acc, desc(a + s * 128 * KSB + k * 256), desc(b + s * brows * KSB + k * 256), j > 0, tbase + SF);
    }
}

// one CTA pair: C (256 x N_) parity of A (256 x K) * B^T (N_ x K); CTA r: A rows 128r.., B rows 112r..
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_pair_check(const uint8_t* A8, const uint8_t* B8, uint32_t* C) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    load_ops(sm, A8 + size_t(rank) * 128 * 512, B8 + size_t(rank) * (N_ / 2) * 512, 128, N_ / 2);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tbase_s)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tbase_s;
    fill_scales(tbase, warp);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (rank == 0 && threadIdx.x == 0) {
        issue_k<256>(tbase, 0, su32(sm), su32(sm) + 128 * 512, N_ / 2);
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                         su32(&mbar)),
                     "h"(static_cast<uint16_t>(3)));
    }
    wait_parity(&mbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int row = rank * 128 + warp * 32 + lane;
    for (int cc = 0; cc < N_ / 32; ++cc) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
              "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tbase + (uint32_t(warp * 32) << 16) + cc * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        uint32_t bits = 0;
        for (int j = 0; j < 32; ++j) bits |= (__float_as_uint(__uint_as_float(v[j]) + 8388608.0f) & 1u) << j;
        C[row * (N_ / 32) + cc] = bits;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
}

// MMA-only rate: random operands resident in smem, iters x 16 MMAs, one commit at the end
template <int M, int READERS>
__global__ void __launch_bounds__(256, 1) k_peak(int iters, int* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase_s;
    const int warp = threadIdx.x >> 5;
    constexpr int brows = M == 256 ? N_ / 2 : N_;
    const uint32_t rank = M == 256 ? cluster_rank() : 0;
    for (int i = threadIdx.x; i < (128 + brows) * 512 / 16; i += blockDim.x) {
        uint32_t h = (i + 1 + 7919 * rank) * 0x9E3779B9u, w[4];
        for (int k = 0; k < 4; ++k) {
            h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
            uint32_t x = 0;
            for (int b = 0; b < 8; ++b) x |= ((h >> b) & 1u) << (4 * b + 1);
            w[k] = x;
        }
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (warp == 0) {
        if (M == 256) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tbase_s)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tbase_s)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tbase_s;
    fill_scales(tbase, warp);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    if (M == 256) cluster_sync();
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (READERS && warp >= 4) {  // epilogue-like TMEM reads of the lane quarter warp & 3, as fast as possible
        uint32_t acc = 0;
        while (!done) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                  "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
                  "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                  "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(tbase + (uint32_t((warp & 3) * 32) << 16) + 2 * N_ - 32 * ((acc & 3) + 1)));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            for (int i = 0; i < 32; ++i) acc += v[i];
        }
        if (acc == 12345u) *sink = acc;
    }
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t a = su32(sm), b = a + 128 * 512;
        for (int it = 0; it < iters; ++it) issue_k<M>(tbase, (it & 1) ? N_ : 0, a, b, brows);
        if (M == 256)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                             su32(&mbar)),
                         "h"(static_cast<uint16_t>(3)));
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&mbar)));
    }
    if (warp < 4) {
        wait_parity(&mbar, 0);
        if (threadIdx.x == 0) done = 1;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tbase));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (threadIdx.x == 0 && v == 12345u) *sink = v;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    if (M == 256) cluster_sync();
    else __syncthreads();
    if (warp == 0) {
        if (M == 256) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
    }
}

int main() {
    constexpr int K = 1024, M = 256;
    std::vector<uint8_t> A(size_t(M) * K), B(size_t(N_) * K);
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
    for (auto& x : A) x = rnd() & 1;
    for (auto& x : B) x = rnd() & 1;
    auto nib = [&](const std::vector<uint8_t>& bits, int rows) {
        std::vector<uint8_t> o(size_t(rows) * K / 2, 0);
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < K; ++k)
                if (bits[size_t(r) * K + k]) o[size_t(r) * (K / 2) + k / 2] |= uint8_t(0x2 << (4 * (k & 1)));
        return o;
    };
    std::vector<uint8_t> A4 = nib(A, M), B4 = nib(B, N_);
    uint8_t *dA, *dB;
    uint32_t* dC;
    CK(cudaMalloc(&dA, A4.size()));
    CK(cudaMalloc(&dB, B4.size()));
    CK(cudaMalloc(&dC, size_t(M) * N_ / 8));
    CK(cudaMemcpy(dA, A4.data(), A4.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B4.data(), B4.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0, size_t(M) * N_ / 8));
    const int smem_pair = (128 + N_ / 2) * 512;
    CK(cudaFuncSetAttribute(k_pair_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pair));
    k_pair_check<<<2, 128, smem_pair>>>(dA, dB, dC);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> C(size_t(M) * N_ / 32);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N_; ++j) {
            int acc = 0;
            for (int k = 0; k < K; ++k) acc += A[size_t(i) * K + k] & B[size_t(j) * K + k];
            bad += ((C[size_t(i) * (N_ / 32) + j / 32] >> (j % 32)) & 1) != (acc & 1);
        }
    printf("pair check 256x%d K=%d (CTA r: A rows 128r.., B rows %dr..): %ld mismatches of %d\n", N_, K, N_ / 2, bad, M * N_);

    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int* sink;
    CK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, int smem, const char* name, int cl) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int iters = 4000;
        auto launch = [&](int it) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nsm);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, kern, it, sink));
        };
        launch(10);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            launch(iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            const double macs = double(nsm) * iters * 16 * 128.0 * N_ * 64.0;  // per SM: 128 rows x N x 64 per MMA
            printf("%s: %.3f ms, %.2f P bit-op/s (%d SMs)\n", name, t, 2 * macs / (t / 1e3) / 1e15, nsm);
        }
    };
    run(k_peak<128, 0>, (128 + N_) * 512, "1-SM  M=128 N=224 (no drain)", 1);
    run(k_peak<128, 1>, (128 + N_) * 512, "1-SM  M=128 N=224 + TMEM readers", 1);
    run(k_peak<256, 0>, (128 + N_ / 2) * 512, "pair  M=256 N=224 (cta_group::2)", 2);
    run(k_peak<256, 1>, (128 + N_ / 2) * 512, "pair  M=256 N=224 + TMEM readers", 2);
    return bad != 0;
}
