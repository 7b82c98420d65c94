// Prototype: GF(2) product C ^= parity(A * B^T) with tcgen05.mma kind::mxf4 (E2M1
// operands, UE8M0 block-32 scales all 1.0): a set bit becomes the fp4 value 1.0
// (nibble 0x2), the fp32 accumulator holds the exact AND-count (<= K <= 2^24) and its
// parity is the GF(2) result.  Both operands K-major (the only major E2M1 allows):
// A8: M rows x K/2 bytes, B8: N rows x K/2 bytes (row n = column n of the product).
// One CTA (256 threads) per 128 x 256 tile; K in stages of 256 elements (128 B per
// row), cp.async into the canonical no-swizzle layout; accumulators + scales in TMEM.
// usage: umma_f4 [M N K]   -> correctness on a sample + Tbit-op/s, then the MMA-only peak
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int BM = 128, BN = 256, KS = 256, KSB = KS / 2, STAGES = 4, NT = 256;
constexpr int A_STAGE = BM * KSB;           // 16 KB
constexpr int B_STAGE = BN * KSB;           // 32 KB
constexpr uint32_t SF_COL = 256;            // scale factors: TMEM columns 256..319, all bytes 0x7F (2^0)
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | (1u << 23) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t((addr >> 4) & 0x3FFF)) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
           (uint64_t(1) << 46);
}
__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
template <uint32_t ID = IDESC>
__device__ __forceinline__ void mma_f4(uint32_t tc, uint64_t da, uint64_t db, uint32_t acc, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tc),
        "l"(da), "l"(db), "r"(ID), "r"(acc), "r"(tsf), "r"(tsf + 32));
}
__device__ __forceinline__ void tmem_setup(uint32_t* tmem_base_smem, int warp) {
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_base_smem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
}
__device__ __forceinline__ void fill_scales(uint32_t tbase, int warp) {
    if (warp < 4) {  // warp w owns TMEM lanes 32w..32w+31
        const uint32_t v = 0x7F7F7F7Fu;
        for (int c = 0; c < 128; c += 8) {  // columns 256..319 and 448..511
            const uint32_t ta = tbase + (uint32_t(warp * 32) << 16) + (c < 64 ? SF_COL + c : 448 + c - 64);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta), "r"(v), "r"(v),
                         "r"(v), "r"(v), "r"(v), "r"(v), "r"(v), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
}

__global__ void __launch_bounds__(NT, 1) k_gf2_f4(const uint8_t* A8, const uint8_t* B8, uint32_t* C, int M, int N, int K) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;
    uint8_t* sB = sm + STAGES * A_STAGE;
    __shared__ uint64_t mbar[STAGES];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int KB = K / 2;

    tmem_setup(&tmem_base, warp);
    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tmem_base;
    fill_scales(tbase, warp);
    asm volatile("tcgen05.fence::before_thread_sync;\n");

    auto load_stage = [&](int st, int kb0) {
        const uint32_t a = smem_u32(sA + st * A_STAGE), b = smem_u32(sB + st * B_STAGE);
        // rows x (KSB/16) chunks of 16 B; addr(r,kc) = (r/8)*SBO + kc*128 + (r%8)*16
        for (int i = tid; i < BM * (KSB / 16); i += NT) {
            const int r8 = i & 7, kc = (i >> 3) % (KSB / 16), rg = (i >> 3) / (KSB / 16);
            cp16(a + rg * ((KSB / 16) * 128) + kc * 128 + r8 * 16, A8 + size_t(m0 + rg * 8 + r8) * KB + kb0 + kc * 16);
        }
        for (int i = tid; i < BN * (KSB / 16); i += NT) {
            const int r8 = i & 7, kc = (i >> 3) % (KSB / 16), rg = (i >> 3) / (KSB / 16);
            cp16(b + rg * ((KSB / 16) * 128) + kc * 128 + r8 * 16, B8 + size_t(n0 + rg * 8 + r8) * KB + kb0 + kc * 16);
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
        if (s < nst) load_stage(s, s * KSB);
        else asm volatile("cp.async.commit_group;\n");
    }
    for (int s = 0; s < nst; ++s) {
        const int sp = s + STAGES - 1;
        if (sp < nst) {
            if (s >= 1) wait_mbar((s - 1) % STAGES, ((s - 1) / STAGES) & 1);
            load_stage(sp % STAGES, sp * KSB);
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
            for (int j = 0; j < KS / 64; ++j) {  // K = 64 elements = 32 B = 2 core matrices per MMA
                const uint64_t da = desc(a + j * 2 * 128, 128, (KSB / 16) * 128);
                const uint64_t db = desc(b + j * 2 * 128, 128, (KSB / 16) * 128);
                mma_f4(tbase, da, db, (s > 0 || j > 0) ? 1u : 0u, tbase + SF_COL);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar[st])));
        }
    }
    wait_mbar((nst - 1) % STAGES, ((nst - 1) / STAGES) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
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
        for (int j = 0; j < 32; ++j) bits |= (__float_as_uint(__uint_as_float(v[j]) + 8388608.0f) & 1u) << j;
        if (row < M) C[size_t(row) * (N / 32) + (n0 / 32) + cc] ^= bits;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
}

// MMA issue rate with smem-resident operands: `iters` x (K/64 MMAs of 128x256x64),
// one commit + wait per group of 16 MMAs; the result is discarded.
// variant bits: 1 = stage layout (4 K-stages of 256 elements, SBO 1024 B, as the Schur
// kernel), 2 = one extra commit per 4 MMAs (to a second mbarrier, never waited on),
// 4 = accumulator alternates between TMEM columns 0 and PN
template <int PN>
__global__ void __launch_bounds__(128, 1) k_f4_peak(int iters, int* sink, int mode, int variant = 0) {
    constexpr uint32_t ID = (1u << 7) | (1u << 10) | (1u << 23) | (uint32_t(PN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t mbar, mbar2;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    // operand data: mode 0 sparse pattern, 1 random bits (E2M1 0/1.0 per nibble), 2 all ones
    for (int i = tid; i < (BM + BN) * 512 / 16; i += 128) {
        uint32_t h = (i + 1) * 0x9E3779B9u;
        uint4 v = make_uint4(0x22222222u, 0, 0x2u, 0);
        if (mode == 2) v = make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u);
        if (mode == 1) {
            uint32_t w[4];
            for (int k = 0; k < 4; ++k) {
                h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
                uint32_t x = 0;
                for (int b = 0; b < 8; ++b) x |= ((h >> b) & 1u) << (4 * b + 1);
                w[k] = x;
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        reinterpret_cast<uint4*>(sm)[i] = v;
    }
    tmem_setup(&tmem_base, warp);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar2)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tmem_base;
    fill_scales(tbase, warp);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    __shared__ volatile int done;
    if (tid == 0) done = 0;
    __syncthreads();
    if (warp > 0 && (variant & 24)) {  // 8: warps 1-3 spin on an mbarrier; 16: they stream TMEM reads
        uint32_t sink2 = 0;
        while (!done) {
            if (variant & 8) {
                uint32_t ok;
                asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}\n"
                             : "=r"(ok) : "r"(smem_u32(&mbar2)));
                sink2 += ok;
            } else {
                uint32_t v[32];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                      "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                      "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(tbase + (uint32_t(warp * 32) << 16) + 320));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                for (int i = 0; i < 32; ++i) sink2 += v[i];
            }
        }
        if (sink2 == 12345) *sink = sink2;
    }
    if (tid == 0) {
        const uint32_t a = smem_u32(sm), b = a + BM * 512;
        for (int it = 0; it < iters; ++it) {
            // 4: alternate accumulators 0 / PN; 32: scale factors at column 448; 64: accumulator at column 224
            const uint32_t acc = (variant & 4) ? ((it & 1) ? tbase + PN : tbase) : (variant & 64) ? tbase + 224 : tbase;
            const uint32_t sf = tbase + ((variant & 32) ? 448 : SF_COL);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                uint64_t da, db;
                if (variant & 1) {  // stage s = j / 4 of 16 KB (A) / PN*128 B (B), K-step j % 4 within it
                    da = desc(a + (j >> 2) * 16384 + (j & 3) * 256, 128, 1024);
                    db = desc(b + (j >> 2) * (PN * 128) + (j & 3) * 256, 128, 1024);
                } else {
                    da = desc(a + j * 2 * 128, 128, 32 * 128);
                    db = desc(b + j * 2 * 128, 128, 32 * 128);
                }
                mma_f4<ID>(acc, da, db, j > 0 ? 1u : 0u, sf);
                if ((variant & 2) && (j & 3) == 3)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar2)));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
            asm volatile(
                "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&mbar)), "r"(it & 1));
        }
        done = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tbase));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (threadIdx.x == 0) *sink = v;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
}

int main(int argc, char** argv) {
    const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 512, K = argc > 3 ? atoi(argv[3]) : 1024;
    std::vector<uint8_t> A(size_t(M) * K), B(size_t(N) * K);  // bits, B row n = product column n
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
    std::vector<uint8_t> A4 = nib(A, M), B4 = nib(B, N);
    uint8_t *dA, *dB;
    uint32_t* dC;
    CK(cudaMalloc(&dA, A4.size()));
    CK(cudaMalloc(&dB, B4.size()));
    CK(cudaMalloc(&dC, size_t(M) * N / 8));
    CK(cudaMemcpy(dA, A4.data(), A4.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B4.data(), B4.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0, size_t(M) * N / 8));
    const size_t smem = STAGES * (A_STAGE + B_STAGE);
    CK(cudaFuncSetAttribute(k_gf2_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 grid(N / BN, M / BM);
    k_gf2_f4<<<grid, NT, smem>>>(dA, dB, dC, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> C(size_t(M) * N / 32);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0, checked = 0;
    for (int i = 0; i < M; i += (M > 512 ? 37 : 1)) {
        for (int j = 0; j < N; ++j) {
            int acc = 0;
            for (int k = 0; k < K; ++k) acc += A[size_t(i) * K + k] & B[size_t(j) * K + k];
            const int got = (C[size_t(i) * (N / 32) + j / 32] >> (j % 32)) & 1;
            bad += got != (acc & 1);
            ++checked;
        }
    }
    printf("M=%d N=%d K=%d: checked %ld bits, %ld mismatches\n", M, N, K, checked, bad);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) k_gf2_f4<<<grid, NT, smem>>>(dA, dB, dC, M, N, K);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int it = 0; it < reps; ++it) k_gf2_f4<<<grid, NT, smem>>>(dA, dB, dC, M, N, K);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("load+mma kernel: %.3f ms per launch, %.1f Tbit-op/s\n", ms / reps, 2.0 * M * N * double(K) * reps / (ms / 1e3) / 1e12);

    int* sink;
    CK(cudaMalloc(&sink, 4));
    const size_t psmem = (BM + BN) * 512;
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    auto peak = [&](auto kern, int pn, int mode, int variant = 0) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(psmem)));
        const int iters = 4000;
        kern<<<nsm, 128, psmem>>>(10, sink, mode, variant);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        kern<<<nsm, 128, psmem>>>(iters, sink, mode, variant);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float t;
        cudaEventElapsedTime(&t, e0, e1);
        const double macs = double(nsm) * iters * 16 * BM * pn * 64.0;
        printf("MMA-only N=%d var=%d data=%s: %.3f ms, %.2f P MAC/s = %.2f P bit-op/s\n", pn, variant,
               mode == 0 ? "sparse" : mode == 1 ? "random" : "ones", t, macs / (t / 1e3) / 1e15, 2 * macs / (t / 1e3) / 1e15);
    };
    for (int v : {0, 32, 96, 36, 37, 39})
        peak(k_f4_peak<224>, 224, 1, v);
    return bad != 0;
}
