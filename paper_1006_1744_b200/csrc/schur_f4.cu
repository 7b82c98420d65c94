// Schur complement C ^= L21 * U12 over GF(2) on the 5th-generation tensor cores.
//
// The same product as k_table_apply (addmul_impl, proj/src/mul.cpp:21-68, with the
// panel's raw-column -> pivot-row map of pls_recursive's update), computed as an
// integer count: a set bit becomes the E2M1 value 1.0 (nibble 0x2), a block-scaled
// tcgen05.mma kind::mxf4 (all UE8M0 scales 2^0) accumulates the exact AND-count of
// each C entry in fp32 (<= K = 1024 < 2^24), and the count's parity is the GF(2)
// sum.  The accumulator starts at 2^23, so the parity is bit 0 of the fp32 word.
//
// Data flow per panel (all device-side, inside the PLS graph):
//   k_f4_expand_a: the coefficient bits of every row below the panel's pivots (A =
//     L21, K-major already) -> nibbles in the canonical no-swizzle K-major layout,
//     one 16 KB block per (128-row tile, 256-K stage): a tile stage is one bulk copy.
//   k_f4_expand_b: the pivot rows U12 gathered by the raw-column map (brow), 32x32
//     bit blocks transposed by warp shuffles (the MMA wants B K-major too) and
//     expanded; one 32 KB block per (256-column tile, K stage).
//   k_schur_f4: persistent, one CTA per SM.  A CTA claims chunks of 16 consecutive
//     tiles (column-tile major, so the CTA's B tile -- 128 KB, the whole K -- stays in
//     SMEM across a chunk and is reloaded stage by stage while the last tile of the
//     old column still computes).  Warp 1 streams A stages through a 4-deep ring
//     (cp.async.bulk + mbarrier transaction counts), one thread of warp 0 issues 4
//     MMAs of 128x256x64 per stage into a 256-column TMEM accumulator, and 16
//     epilogue warps (4 per TMEM lane quarter, 64 columns each) read the counts,
//     re-arm the accumulator with 2^23, release it, pack 64 parities into a word by
//     funnel shifts and XOR it into C.  Tiles and the chunk queue are data dependent
//     (the row count comes from the panel snapshot), so no host sync is needed.
#include <cstdint>
#include <cstdlib>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kFM = 128, kFN = 256, kFKS = 256;   // tile rows / cols, K elements per stage
constexpr int kFAStage = kFM * kFKS / 2;          // 16 KB of nibbles
constexpr int kFBStage = kFN * kFKS / 2;          // 32 KB
constexpr int kFMaxStages = 4;                    // K <= 1024
constexpr int kFRing = 4;                         // A stages in flight
constexpr int kFChunk = 16;                       // tiles per claimed chunk
constexpr int kFQ = 8;                            // chunk-id broadcast ring
constexpr int kFThreads = 640;                    // warp 0 MMA, warp 1 loads, warps 4..19 epilogue
constexpr int kFEpiWarps = 16;
constexpr uint32_t kFSfCol = 256;                 // TMEM columns 256..319: scale factors (all 0x7F)
constexpr uint32_t kFIdesc = (1u << 7) | (1u << 10) | (1u << 23) | (static_cast<uint32_t>(kFN >> 3) << 17) |
                             (static_cast<uint32_t>(kFM >> 4) << 24);  // E2M1 x E2M1, UE8M0, K-major, 128x256
constexpr size_t kFSmem = static_cast<size_t>(kFMaxStages) * kFBStage + static_cast<size_t>(kFRing) * kFAStage;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// canonical no-swizzle K-major operand: 8-row x 16-byte core matrices, LBO = 128 B
// between K-adjacent ones, SBO = 1024 B between row groups (a stage is 8 chunks wide)
__device__ __forceinline__ uint64_t f4_desc(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(128 >> 4) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mb_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(su32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// 8 bits -> 8 nibbles holding 0x2 (E2M1 1.0) per set bit, bit i -> nibble i
__device__ __forceinline__ uint32_t spread8(uint32_t x) {
    x &= 0xffu;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    x = (x | (x << 3)) & 0x11111111u;
    return x << 1;
}
__device__ __forceinline__ uint4 spread32(uint32_t x) {
    return make_uint4(spread8(x), spread8(x >> 8), spread8(x >> 16), spread8(x >> 24));
}

// lane l holds row l (bit c = column c) -> lane l holds column l (bit r = row r)
__device__ __forceinline__ uint32_t transpose32(uint32_t v, int lane) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v, s);
        v = (lane & s) ? ((v & ~m) | ((o >> s) & m)) : ((v & m) | ((o << s) & ~m));
    }
    return v;
}

}  // namespace

// A = coefficient bits [aw0*64, aw0*64 + kbits) of rows r0 + i, r0 = rk[0] + rk[1]
__global__ void __launch_bounds__(256) k_f4_expand_a(Mat A, int64_t aw0, int64_t kbits, const int64_t* rk, int64_t m,
                                                     uint8_t* __restrict__ Ax, int nst) {
    const int64_t r0 = rk[0] + rk[1];
    const int64_t rows = m - r0;
    if (rows <= 0) return;
    const int64_t nrt = (rows + kFM - 1) / kFM;
    const int64_t total = nrt * nst * 1024;  // 16-byte output chunks
    for (int64_t idx = blockIdx.x * 256ll + threadIdx.x; idx < total; idx += static_cast<int64_t>(gridDim.x) * 256) {
        const int r8 = static_cast<int>(idx & 7), kc = static_cast<int>((idx >> 3) & 7), rg = static_cast<int>((idx >> 6) & 15);
        const int64_t blk = idx >> 10;
        const int s = static_cast<int>(blk % nst);
        const int64_t rt = blk / nst;
        const int64_t row = rt * kFM + rg * 8 + r8;
        const int64_t j0 = static_cast<int64_t>(s) * kFKS + kc * 32;
        uint32_t x = 0;
        if (row < rows && j0 < kbits) {
            x = reinterpret_cast<const uint32_t*>(A.w + (r0 + row) * A.stride + aw0)[j0 >> 5];
            if (kbits - j0 < 32) x &= (1u << (kbits - j0)) - 1u;
        }
        reinterpret_cast<uint4*>(Ax)[idx] = spread32(x);  // offset = ((rt*nst + s) * 1024 + rg*64 + kc*8 + r8) * 16
    }
}

// B^T: element (n, j) = bit (n) of pivot row brow[j] over words [cw0, cw1) of U
__global__ void __launch_bounds__(256) k_f4_expand_b(Mat U, const int64_t* __restrict__ brow, int64_t kbits, int64_t cw0,
                                                     int64_t cw1, uint8_t* __restrict__ Bx, int nst) {
    const int lane = threadIdx.x & 31;
    const int64_t nct = (cw1 - cw0 + 3) / 4;
    const int64_t tasks = nct * nst * 8 * 4;  // (tile, stage, 32-K block, 64-column word)
    for (int64_t w = (blockIdx.x * 256ll + threadIdx.x) >> 5; w < tasks; w += (static_cast<int64_t>(gridDim.x) * 256) >> 5) {
        const int wd = static_cast<int>(w & 3), kq = static_cast<int>((w >> 2) & 7);
        const int64_t blk = w >> 5;
        const int s = static_cast<int>(blk % nst);
        const int64_t ct = blk / nst;
        const int64_t j = static_cast<int64_t>(s) * kFKS + kq * 32 + lane;
        const int64_t word = cw0 + ct * 4 + wd;
        uint64_t v = 0;
        if (j < kbits && word < cw1) {
            const int64_t br = brow[j];
            if (br >= 0) v = U.w[br * U.stride + word];
        }
        uint8_t* base = Bx + (ct * nst + s) * kFBStage + kq * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t t = transpose32(static_cast<uint32_t>(v >> (32 * h)), lane);
            const int n = wd * 64 + h * 32 + lane;  // column within the tile
            *reinterpret_cast<uint4*>(base + (n >> 3) * 1024 + (n & 7) * 16) = spread32(t);
        }
    }
}

__global__ void __launch_bounds__(kFThreads, 1)
k_schur_f4(Mat C, int64_t cw0, int64_t cw1, const int64_t* __restrict__ rk, int64_t m, const uint8_t* __restrict__ Ax,
           const uint8_t* __restrict__ Bx, int nst, unsigned* __restrict__ claim) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* sB = smem;                               // [nst][32 KB]
    uint8_t* sA = smem + kFMaxStages * kFBStage;      // ring [kFRing][16 KB]
    __shared__ __align__(8) uint64_t a_full[kFRing], a_empty[kFRing], b_full[kFMaxStages], b_empty[kFMaxStages];
    __shared__ __align__(8) uint64_t acc_full, acc_empty, q_full[kFQ], q_empty[kFQ];
    __shared__ int64_t q_chunk[kFQ];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t r0 = rk[0] + rk[1];
    const int64_t rows = m - r0;
    if (rows <= 0 || cw1 <= cw0) return;
    const int64_t nrt = (rows + kFM - 1) / kFM, nct = (cw1 - cw0 + 3) / 4;
    const int64_t T = nrt * nct;
    const int64_t nchunks = (T + kFChunk - 1) / kFChunk;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        for (int i = 0; i < kFRing; ++i) {
            mb_init(&a_full[i], 1);
            mb_init(&a_empty[i], 1);
        }
        for (int i = 0; i < kFMaxStages; ++i) {
            mb_init(&b_full[i], 1);
            mb_init(&b_empty[i], 1);
        }
        mb_init(&acc_full, 1);
        mb_init(&acc_empty, kFEpiWarps);
        for (int i = 0; i < kFQ; ++i) {
            mb_init(&q_full[i], 1);
            mb_init(&q_empty[i], 1 + kFEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tbase = tmem_base;

    if (warp == 1) {
        if (lane == 0) {  // ---------------- loads + chunk claims ----------------
            int64_t cur_ct = -1, u = 0, tiles = 0, bu = 0;
            for (int64_t qi = 0;; ++qi) {
                const int slot = static_cast<int>(qi % kFQ);
                if (qi >= kFQ) mb_wait(&q_empty[slot], static_cast<uint32_t>((qi / kFQ - 1) & 1));
                const int64_t ch = static_cast<int64_t>(atomicAdd(claim, 1u));
                q_chunk[slot] = ch < nchunks ? ch : -1;
                mb_arrive(&q_full[slot]);  // release: the consumers read q_chunk after the wait
                if (ch >= nchunks) break;
                const int64_t t1 = (ch + 1) * kFChunk < T ? (ch + 1) * kFChunk : T;
                for (int64_t t = ch * kFChunk; t < t1; ++t, ++tiles) {
                    const int64_t ct = t / nrt, rt = t % nrt;
                    if (ct != cur_ct) {  // new B tile, stage by stage behind the MMAs of the old one
                        for (int s = 0; s < nst; ++s) {
                            if (tiles > 0) mb_wait(&b_empty[s], static_cast<uint32_t>((tiles - 1) & 1));
                            mb_expect_tx(&b_full[s], kFBStage);
                            bulk_g2s(sB + s * kFBStage, Bx + (ct * nst + s) * kFBStage, kFBStage, &b_full[s]);
                        }
                        cur_ct = ct;
                        ++bu;
                    }
                    for (int s = 0; s < nst; ++s, ++u) {
                        const int sl = static_cast<int>(u % kFRing);
                        const int64_t f = u / kFRing;
                        if (f > 0) mb_wait(&a_empty[sl], static_cast<uint32_t>((f - 1) & 1));
                        mb_expect_tx(&a_full[sl], kFAStage);
                        bulk_g2s(sA + sl * kFAStage, Ax + (rt * nst + s) * kFAStage, kFAStage, &a_full[sl]);
                    }
                }
            }
            (void)bu;
        }
    } else if (warp == 0) {
        if (lane == 0) {  // ---------------- MMA issue ----------------
            int64_t cur_ct = -1, u = 0, tiles = 0, bu = 0;
            for (int64_t qi = 0;; ++qi) {
                const int slot = static_cast<int>(qi % kFQ);
                mb_wait(&q_full[slot], static_cast<uint32_t>((qi / kFQ) & 1));
                const int64_t ch = q_chunk[slot];
                mb_arrive(&q_empty[slot]);
                if (ch < 0) break;
                const int64_t t1 = (ch + 1) * kFChunk < T ? (ch + 1) * kFChunk : T;
                for (int64_t t = ch * kFChunk; t < t1; ++t, ++tiles) {
                    const int64_t ct = t / nrt;
                    const bool newb = ct != cur_ct;
                    if (newb) {
                        cur_ct = ct;
                        ++bu;
                    }
                    mb_wait(&acc_empty, static_cast<uint32_t>(tiles & 1));
                    tc_after();
                    for (int s = 0; s < nst; ++s, ++u) {
                        if (newb) mb_wait(&b_full[s], static_cast<uint32_t>((bu - 1) & 1));
                        const int sl = static_cast<int>(u % kFRing);
                        mb_wait(&a_full[sl], static_cast<uint32_t>((u / kFRing) & 1));
                        tc_after();
                        const uint32_t a = su32(sA + sl * kFAStage), b = su32(sB + s * kFBStage);
#pragma unroll
                        for (int j = 0; j < kFKS / 64; ++j) {
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], "
                                "p;\n\t}\n" ::"r"(tbase),
                                "l"(f4_desc(a + j * 256)), "l"(f4_desc(b + j * 256)), "r"(kFIdesc), "r"(tbase + kFSfCol),
                                "r"(tbase + kFSfCol + 32));
                        }
                        mma_commit(&a_empty[sl]);  // A stage free once these MMAs are done
                        mma_commit(&b_empty[s]);   // (phase per tile) B stage s reusable
                    }
                    mma_commit(&acc_full);
                }
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue ----------------
        const int q = warp & 3, h = (warp - 4) >> 2;
        const uint32_t tl = tbase + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t bias = 0x4B000000u;  // 2^23
        if (h == 0) {  // scale factors: every byte 0x7F = 2^0
            const uint32_t v = 0x7F7F7F7Fu;
            for (int c = 0; c < 64; c += 8)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(tl + kFSfCol + c),
                             "r"(v));
        }
        auto arm = [&]() {  // accumulator columns of this warp := 2^23
#pragma unroll
            for (int c = 0; c < 64; c += 16)
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                        tl + h * 64 + c),
                    "r"(bias));
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            tc_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&acc_empty);
        };
        arm();
        int64_t tiles = 0;
        for (int64_t qi = 0;; ++qi) {
            const int slot = static_cast<int>(qi % kFQ);
            mb_wait(&q_full[slot], static_cast<uint32_t>((qi / kFQ) & 1));
            const int64_t ch = q_chunk[slot];
            __syncwarp();
            if (lane == 0) mb_arrive(&q_empty[slot]);
            if (ch < 0) break;
            const int64_t t1 = (ch + 1) * kFChunk < T ? (ch + 1) * kFChunk : T;
            for (int64_t t = ch * kFChunk; t < t1; ++t, ++tiles) {
                const int64_t ct = t / nrt, rt = t % nrt;
                mb_wait(&acc_full, static_cast<uint32_t>(tiles & 1));
                tc_after();
                uint32_t half[2];
#pragma unroll
                for (int c = 0; c < 2; ++c) {  // 32 columns at a time: fewer live registers
                    uint32_t v[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(tl + h * 64 + c * 32));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    uint32_t x = 0;
#pragma unroll
                    for (int i = 0; i < 32; ++i) x = __funnelshift_r(x, v[i], 1);
                    half[c] = x;
                }
                arm();
                const uint32_t lo = half[0], hi = half[1];
                const int64_t row = r0 + rt * kFM + q * 32 + lane;
                const int64_t word = cw0 + ct * 4 + h;
                if (row < m && word < cw1) C.w[row * C.stride + word] ^= static_cast<uint64_t>(lo) | (static_cast<uint64_t>(hi) << 32);
            }
        }
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
}

size_t schur_f4_a_bytes(int64_t rows) { return static_cast<size_t>((rows + kFM - 1) / kFM) * kFMaxStages * kFAStage; }
size_t schur_f4_b_bytes(int64_t words) { return static_cast<size_t>((words + 3) / 4) * kFMaxStages * kFBStage; }

// K is always padded to kFMaxStages stages (zero nibbles): the B ring then spans exactly
// one tile, which the loader's B-reload waits rely on (one mbarrier phase per tile)
void launch_schur_f4_expand_a(cudaStream_t s, const Mat& A, int64_t aw0, int64_t kbits, const int64_t* rk, uint8_t* Ax,
                              int nsm) {
    const int nst = kFMaxStages;
    k_f4_expand_a<<<nsm * 8, 256, 0, s>>>(A, aw0, kbits, rk, A.m, Ax, nst);
}

void launch_schur_f4(cudaStream_t s, const Mat& C, int64_t cw0, int64_t cw1, const int64_t* rk, const int64_t* brow,
                     int64_t kbits, const uint8_t* Ax, uint8_t* Bx, unsigned* claim, int nsm) {
    if (cw1 <= cw0) return;
    const int nst = kFMaxStages;
    k_f4_expand_b<<<nsm * 8, 256, 0, s>>>(C, brow, kbits, cw0, cw1, Bx, nst);
    cudaMemsetAsync(claim, 0, sizeof(unsigned), s);
    k_schur_f4<<<nsm, kFThreads, kFSmem, s>>>(C, cw0, cw1, rk, C.m, Ax, Bx, nst, claim);
}

void setup_schur_f4_kernels() {
    cudaFuncSetAttribute(k_schur_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kFSmem));
}

}  // namespace f2g
