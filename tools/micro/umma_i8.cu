// Prototype: GF(2) product C = parity(A * B) with tcgen05.mma kind::i8.
// A8: M x K bytes (0/1, K-major), B8: K x N bytes (0/1, N-major = MN-major operand).
// One CTA (128 threads) per 128 x 256 tile; K in stages of 128 bytes (4 MMAs of K=32),
// operands staged by cp.async into the canonical no-swizzle layouts; accumulators in TMEM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int BM = 128, BN = 256, KS = 128, STAGES = 4, NT = 256;
constexpr int A_STAGE = BM * KS;           // 16 KB
constexpr int B_STAGE = KS * BN;           // 32 KB
constexpr uint32_t IDESC = (2u << 4) | (1u << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t((addr >> 4) & 0x3FFF)) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
           (uint64_t(1) << 46);
}
__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}

__global__ void __launch_bounds__(NT, 1) k_gf2_umma(const uint8_t* A8, const uint8_t* B8, uint32_t* C, int M, int N, int K) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;
    uint8_t* sB = sm + STAGES * A_STAGE;
    __shared__ uint64_t mbar[STAGES];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tmem_base;

    auto load_stage = [&](int st, int k0) {
        const uint32_t a = smem_u32(sA + st * A_STAGE), b = smem_u32(sB + st * B_STAGE);
        // A: 128 rows x (KS/16) chunks of 16 B; addr(r,kc) = (r/8)*SBO + kc*128 + (r%8)*16.
        // Consecutive lanes fill one 128-B core matrix (conflict-free smem writes).
        for (int i = tid; i < BM * (KS / 16); i += NT) {
            const int r8 = i & 7, kc = (i >> 3) % (KS / 16), rg = (i >> 3) / (KS / 16);
            const int r = rg * 8 + r8;
            cp16(a + rg * ((KS / 16) * 128) + kc * 128 + r8 * 16, A8 + size_t(m0 + r) * K + k0 + kc * 16);
        }
        // B: KS k-rows x (BN/16) chunks of 16 N-bytes; addr(k,nc) = nc*SBO + (k/8)*128 + (k%8)*16
        for (int i = tid; i < KS * (BN / 16); i += NT) {
            const int k8 = i & 7, kg = (i >> 3) % (KS / 8), nc = (i >> 3) / (KS / 8);
            const int k = kg * 8 + k8;
            cp16(b + nc * ((KS / 8) * 128) + kg * 128 + k8 * 16, B8 + size_t(k0 + k) * N + n0 + nc * 16);
        }
        asm volatile("cp.async.commit_group;\n");
    };

    const int nst = K / KS;
    auto wait_mbar = [&](int b, uint32_t parity) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&mbar[b])), "r"(parity));
    };
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nst) load_stage(s, s * KS);
        else asm volatile("cp.async.commit_group;\n");
    }
    for (int s = 0; s < nst; ++s) {
        const int sp = s + STAGES - 1;  // stage to prefetch, into the buffer MMA s-1 used
        if (sp < nst) {
            if (s >= 1) wait_mbar((s - 1) % STAGES, ((s - 1) / STAGES) & 1);
            load_stage(sp % STAGES, sp * KS);
        } else {
            asm volatile("cp.async.commit_group;\n");
        }
        asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 1));
        asm volatile("fence.proxy.async.shared::cta;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (tid == 0) {
            const int st = s % STAGES;
            const uint32_t a = smem_u32(sA + st * A_STAGE), b = smem_u32(sB + st * B_STAGE);
#pragma unroll
            for (int j = 0; j < KS / 32; ++j) {
                const uint64_t da = desc(a + j * 2 * 128, 128, (KS / 16) * 128);
                const uint64_t db = desc(b + j * 4 * 128, 128, (KS / 8) * 128);
                const uint32_t acc = (s > 0 || j > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tbase),
                    "l"(da), "l"(db), "r"(IDESC), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar[st])));
        }
    }
    // all MMAs done: the last commit covers every earlier MMA
    wait_mbar((nst - 1) % STAGES, ((nst - 1) / STAGES) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // epilogue: warp w reads TMEM lanes 32(w%4).. (rows); warps 0-3 take column chunks
    // 0..3, warps 4-7 chunks 4..7
    const int row = m0 + (warp & 3) * 32 + lane;
#pragma unroll 1
    for (int cc = (warp >> 2) * 4; cc < (warp >> 2) * 4 + 4; ++cc) {
        uint32_t v[32];
        const uint32_t taddr = tbase + (uint32_t((warp & 3) * 32) << 16) + cc * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) bits |= (v[j] & 1u) << j;
        if (row < M) C[size_t(row) * (N / 32) + (n0 / 32) + cc] ^= bits;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(256));
}

int main(int argc, char** argv) {
    const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 512, K = argc > 3 ? atoi(argv[3]) : 1024;
    std::vector<uint8_t> A(size_t(M) * K), B(size_t(K) * N);
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
    for (auto& x : A) x = rnd() & 1;
    for (auto& x : B) x = rnd() & 1;
    uint8_t *dA, *dB;
    uint32_t* dC;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dC, size_t(M) * N / 8));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0, size_t(M) * N / 8));
    const size_t smem = STAGES * (A_STAGE + B_STAGE);
    CK(cudaFuncSetAttribute(k_gf2_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 grid(N / BN, M / BM);
    k_gf2_umma<<<grid, NT, smem>>>(dA, dB, dC, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> C(size_t(M) * N / 32);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    // check a sample of rows on the CPU
    long bad = 0, checked = 0;
    for (int i = 0; i < M; i += (M > 512 ? 37 : 1)) {
        for (int j = 0; j < N; ++j) {
            int acc = 0;
            for (int k = 0; k < K; ++k) acc += A[size_t(i) * K + k] & B[size_t(k) * N + j];
            const int got = (C[size_t(i) * (N / 32) + j / 32] >> (j % 32)) & 1;
            bad += got != (acc & 1);
            ++checked;
        }
    }
    printf("M=%d N=%d K=%d: checked %ld bits, %ld mismatches\n", M, N, K, checked, bad);
    // timing
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) k_gf2_umma<<<grid, NT, smem>>>(dA, dB, dC, M, N, K);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int it = 0; it < reps; ++it) k_gf2_umma<<<grid, NT, smem>>>(dA, dB, dC, M, N, K);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * M * N * double(K) * reps;
    printf("time %.3f ms per launch, %.1f Tbit-op/s\n", ms / reps, ops / (ms / 1e3) / 1e12);
    return bad != 0;
}
