// Schur complement C ^= L21 * U12 over GF(2) on the 5th-generation tensor cores.
//
// The same product as k_table_apply (addmul_impl, proj/src/mul.cpp:21-68, with the
// panel's raw-column -> pivot-row map of pls_recursive's update), computed as an
// integer count: a set bit becomes the E2M1 value 1.0 (nibble 0x2), a block-scaled
// tcgen05.mma kind::mxf4 (all UE8M0 scales 2^0) accumulates the exact AND-count of
// each C entry in fp32 (<= K = 1024 < 2^24), and the count's parity is the GF(2)
// sum: bit 0 of the fp32 word of count + 2^23.
//
// Data flow per panel (all device-side, inside the PLS graph):
//   k_f4_expand_a: the coefficient bits of every row below the panel's pivots (A =
//     L21, K-major already) -> nibbles in the canonical no-swizzle K-major layout,
//     one 16 KB block per (128-row tile, 256-K stage): a tile stage is one bulk copy.
//   k_f4_expand_b: the pivot rows U12 gathered by the raw-column map (brow), 32x32
//     bit blocks transposed by warp shuffles (the MMA wants B K-major too) and
//     expanded; one 28 KB block per (224-column tile, K stage).
//   k_schur_f4: persistent, one CTA per SM.  A CTA claims chunks of consecutive tiles
//     (column-tile major, so the CTA's B tile -- 112 KB, the whole K -- stays in SMEM
//     across a chunk and is reloaded stage by stage behind the last MMAs on the old
//     one; chunk size from the launch: k equal chunks of <= 64 tiles per CTA).  Warp 1
//     streams A stages through a 6-deep ring (cp.async.bulk + mbarrier transaction
//     counts); one elected lane of the converged warp 0 issues 4 MMAs of 128x224x64 per
//     stage into one of two TMEM accumulators (2 x 224 columns + 64 scale-factor
//     columns = all 512); 4 epilogue warps (one per TMEM lane quarter) read 32-column
//     groups, release the buffer, pack parities by funnel shifts and XOR them into C
//     with fire-and-forget RED.  Tiles and the chunk queue are data dependent (the row
//     count comes from the panel snapshot), so no host sync is needed.  No runtime
//     switch may sit in the issue, load or epilogue loops: a single one cost 5-9 %.
#include <cstdint>
#include <cstdlib>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kFM = 128, kFN = 224, kFKS = 256;   // tile rows / cols (7 half-words), K elements per stage
constexpr int kFHW = kFN / 32;                    // 32-bit column groups per tile
constexpr int kFAStage = kFM * kFKS / 2;          // 16 KB of nibbles
constexpr int kFBStage = kFN * kFKS / 2;          // 28 KB
constexpr int kFMaxStages = 4;                    // K <= 1024
constexpr int kFRingMax = 6;                      // A stages in flight (template RING <= this)
constexpr int kFQ = 8;                            // chunk-id broadcast ring
// threads: warp 0 MMA, warp 1 loads, warps 2-3 idle, 4 * EPW epilogue warps from warp 4
constexpr int f4_threads(int epw) { return 128 + 128 * epw; }
constexpr uint32_t kFSfCol = 2 * kFN;             // TMEM: accumulators 0..447 (two tiles), scale factors 448..511
constexpr uint32_t kFIdesc = (1u << 7) | (1u << 10) | (1u << 23) | (static_cast<uint32_t>(kFN >> 3) << 17) |
                             (static_cast<uint32_t>(kFM >> 4) << 24);  // E2M1 x E2M1, UE8M0, K-major, 128x224
constexpr size_t f4_smem(int ring) { return static_cast<size_t>(kFMaxStages) * kFBStage + static_cast<size_t>(ring) * kFAStage; }

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

__device__ __forceinline__ int64_t f4_row_shift(const F4Job& jb) { return jb.rk ? jb.rk[0] + jb.rk[1] : 0; }

// A = coefficient bits [aw0*64, aw0*64 + kbits) of rows a_r0 + d + i
__global__ void __launch_bounds__(256) k_f4_expand_a(F4Job jb, uint8_t* __restrict__ Ax, int nst) {
    pdl_wait();
    const int64_t d = f4_row_shift(jb);
    const int64_t rows = jb.rows_end - d;
    if (rows <= 0) return;
    const int64_t nrt = (rows + kFM - 1) / kFM;
    const int64_t total = nrt * nst * 1024;  // 16-byte output chunks
    const uint64_t* abase = jb.A.w + (jb.a_r0 + d) * jb.A.stride + jb.aw0;
    for (int64_t idx = blockIdx.x * 256ll + threadIdx.x; idx < total; idx += static_cast<int64_t>(gridDim.x) * 256) {
        const int r8 = static_cast<int>(idx & 7), kc = static_cast<int>((idx >> 3) & 7), rg = static_cast<int>((idx >> 6) & 15);
        const int64_t blk = idx >> 10;
        const int s = static_cast<int>(blk % nst);
        const int64_t rt = blk / nst;
        const int64_t row = rt * kFM + rg * 8 + r8;
        const int64_t j0 = static_cast<int64_t>(s) * kFKS + kc * 32;
        uint32_t x = 0;
        if (row < rows && j0 < jb.kbits) {
            x = reinterpret_cast<const uint32_t*>(abase + row * jb.A.stride)[j0 >> 5];
            if (jb.kbits - j0 < 32) x &= (1u << (jb.kbits - j0)) - 1u;
        }
        reinterpret_cast<uint4*>(Ax)[idx] = spread32(x);  // offset = ((rt*nst + s) * 1024 + rg*64 + kc*8 + r8) * 16
    }
}

// B^T: element (n, j) = bit n of B row (brow ? brow[j] : b_r0 + j), columns from 32-bit
// half-word 2*bw0 on; a tile is kFHW half-words of C starting at 2*cw0 + ct*kFHW
// (also zeroes the Schur launch's work counter: no memset node between the two kernels)
__global__ void __launch_bounds__(256) k_f4_expand_b(F4Job jb, uint8_t* __restrict__ Bx, int nst, unsigned* claim) {
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) *claim = 0u;
    if (jb.rows_end - f4_row_shift(jb) <= 0) return;  // no rows below the pivots: the product is empty
    const int lane = threadIdx.x & 31;
    const int64_t nhw = 2 * (jb.cw1 - jb.cw0);
    const int64_t nct = (nhw + kFHW - 1) / kFHW;
    const int64_t tasks = nct * nst * 8 * kFHW;  // (tile, stage, 32-K block, half-word)
    for (int64_t w = (blockIdx.x * 256ll + threadIdx.x) >> 5; w < tasks; w += (static_cast<int64_t>(gridDim.x) * 256) >> 5) {
        const int hw = static_cast<int>(w % kFHW);
        const int64_t rest = w / kFHW;
        const int kq = static_cast<int>(rest & 7);
        const int64_t blk = rest >> 3;
        const int s = static_cast<int>(blk % nst);
        const int64_t ct = blk / nst;
        const int64_t j = static_cast<int64_t>(s) * kFKS + kq * 32 + lane;
        const int64_t x = ct * kFHW + hw;  // half-word within the column range
        uint32_t v = 0;
        if (j < jb.kbits && x < nhw) {
            const int64_t br = jb.brow ? jb.brow[j] : jb.b_r0 + j;
            if (br >= 0) v = reinterpret_cast<const uint32_t*>(jb.B.w + br * jb.B.stride + jb.bw0)[x];
        }
        const uint32_t t = transpose32(v, lane);
        const int n = hw * 32 + lane;  // column within the tile
        *reinterpret_cast<uint4*>(Bx + (ct * nst + s) * kFBStage + kq * 128 + (n >> 3) * 1024 + (n & 7) * 16) = spread32(t);
    }
}

// One elected lane of a converged warp issues; the rest of the warp runs the same
// uniform loop (operands stay in uniform registers, no per-MMA lane waterfall).
__device__ __forceinline__ void f4_mma(uint32_t d, uint64_t da, uint64_t db, uint32_t sfa, uint32_t sfb, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %6, [%3], [%4], p;\n\t}\n" ::"r"(d),
        "l"(da), "l"(db), "r"(sfa), "r"(sfb), "r"(accum), "n"(kFIdesc));
}
__device__ __forceinline__ void f4_commit(uint64_t* b) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(su32(b))
        : "memory");
}

// Tile walk shared by the three roles: chunk ch covers tiles [16 ch, 16 ch + 16) of the
// column-major tile order (row tile fastest), so consecutive tiles share the B tile.
struct F4Walk {
    int rt, ct, n;  // current tile, tiles left in the chunk
    __device__ __forceinline__ F4Walk(int64_t ch, int nrt, int64_t T, int chunk) {
        const int64_t t = ch * chunk;
        ct = static_cast<int>(t / nrt);
        rt = static_cast<int>(t - static_cast<int64_t>(ct) * nrt);
        n = static_cast<int>(T - t < chunk ? T - t : chunk);
    }
    __device__ __forceinline__ void next(int nrt) {
        if (++rt == nrt) {
            rt = 0;
            ++ct;
        }
    }
};

template <int kFRing, int EPW>
__global__ void __launch_bounds__(f4_threads(EPW), 1)
k_schur_f4(F4Job jb, const uint8_t* __restrict__ Ax, const uint8_t* __restrict__ Bx, unsigned* __restrict__ claim,
           unsigned long long* tl) {
    pdl_wait();
    constexpr int NST = kFMaxStages;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sB = smem;                        // [NST][28 KB], the whole K of one column tile
    uint8_t* sA = smem + NST * kFBStage;       // ring [kFRing][16 KB] of A stages
    __shared__ __align__(8) uint64_t a_full[kFRing], a_empty[kFRing], b_full[NST], b_empty[NST];
    __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2], q_full[kFQ], q_empty[kFQ];
    __shared__ int64_t q_chunk[kFQ];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t d = f4_row_shift(jb);
    const int64_t rows = jb.rows_end - d;
    const int64_t cw0 = jb.cw0, cw1 = jb.cw1;
    if (rows <= 0 || cw1 <= cw0) return;
    if (tl && tid == 0) atomicMin(tl, gtimer());  // F2_TIMELINE builds: [start, end] of the launch
    const int64_t nhw = 2 * (cw1 - cw0);
    const int nrt = static_cast<int>((rows + kFM - 1) / kFM), nct = static_cast<int>((nhw + kFHW - 1) / kFHW);
    const int64_t T = static_cast<int64_t>(nrt) * nct;
    // chunk: k = ceil(tiles per CTA / cap) chunks per CTA of equal size <= cap (long runs on one
    // B tile, at most one tile of imbalance when the grid divides the work evenly)
    const int64_t per_cta = (T + gridDim.x - 1) / gridDim.x;
    constexpr int cap = 64;
    const int64_t kch = (per_cta + cap - 1) / cap;
    const int chunk = static_cast<int>((T + gridDim.x * kch - 1) / (gridDim.x * kch));
    const int64_t nchunks = (T + chunk - 1) / chunk;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        for (int i = 0; i < kFRing; ++i) {
            mb_init(&a_full[i], 1);
            mb_init(&a_empty[i], 1);
        }
        for (int i = 0; i < NST; ++i) {
            mb_init(&b_full[i], 1);
            mb_init(&b_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mb_init(&acc_full[i], 1);
            mb_init(&acc_empty[i], 4 * EPW);
        }
        for (int i = 0; i < kFQ; ++i) {
            mb_init(&q_full[i], 1);
            mb_init(&q_empty[i], 1 + 4 * EPW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tbase = tmem_base;

    if (warp == 1) {
        if (lane == 0) {  // ---------------- chunk claims + bulk copies ----------------
            int cur_ct = -1;
            uint32_t u = 0, tiles = 0;  // A stages issued, tiles walked
            for (int64_t qi = 0;; ++qi) {
                const int slot = static_cast<int>(qi % kFQ);
                if (qi >= kFQ) mb_wait(&q_empty[slot], static_cast<uint32_t>((qi / kFQ - 1) & 1));
                const int64_t ch = static_cast<int64_t>(atomicAdd(claim, 1u));
                q_chunk[slot] = ch < nchunks ? ch : -1;
                mb_arrive(&q_full[slot]);  // release: the consumers read q_chunk after the wait
                if (ch >= nchunks) break;
                for (F4Walk w(ch, nrt, T, chunk); w.n > 0; --w.n, w.next(nrt), ++tiles) {
                    if (w.ct != cur_ct) {  // new B tile, stage by stage behind the last MMAs on the old one
                        for (int s = 0; s < NST; ++s) {
                            // b_empty[s] completes one phase per tile: wait for the previous tile's
                            // (the current tile cannot have started: its B is not loaded yet)
                            if (tiles > 0) mb_wait(&b_empty[s], (tiles - 1) & 1);
                            mb_expect_tx(&b_full[s], kFBStage);
                            bulk_g2s(sB + s * kFBStage, Bx + (static_cast<int64_t>(w.ct) * NST + s) * kFBStage, kFBStage,
                                     &b_full[s]);
                        }
                        cur_ct = w.ct;
                    }
                    for (int s = 0; s < NST; ++s, ++u) {
                        const uint32_t sl = u % kFRing, f = u / kFRing;
                        if (f > 0) mb_wait(&a_empty[sl], (f - 1) & 1);
                        mb_expect_tx(&a_full[sl], kFAStage);
                        bulk_g2s(sA + sl * kFAStage, Ax + (static_cast<int64_t>(w.rt) * NST + s) * kFAStage, kFAStage,
                                 &a_full[sl]);
                    }
                }
            }
        }
    } else if (warp == 0) {  // ---------------- MMA issue (whole warp, one elected lane) ----------------
        // descriptor bases: a K step of 64 elements is 2 core matrices = 256 B = 16 in the address field
        uint64_t da0[kFRing], db0[NST];
#pragma unroll
        for (int i = 0; i < kFRing; ++i) da0[i] = f4_desc(su32(sA + i * kFAStage));
#pragma unroll
        for (int i = 0; i < NST; ++i) db0[i] = f4_desc(su32(sB + i * kFBStage));
        const uint32_t sfa = tbase + kFSfCol, sfb = tbase + kFSfCol + 32;
        int cur_ct = -1;
        uint32_t u = 0, tiles = 0, bu = 0;
        for (int64_t qi = 0;; ++qi) {
            const int slot = static_cast<int>(qi % kFQ);
            mb_wait(&q_full[slot], static_cast<uint32_t>((qi / kFQ) & 1));
            const int64_t ch = q_chunk[slot];
            __syncwarp();
            if (lane == 0) mb_arrive(&q_empty[slot]);
            if (ch < 0) break;
            for (F4Walk w(ch, nrt, T, chunk); w.n > 0; --w.n, w.next(nrt), ++tiles) {
                const bool newb = w.ct != cur_ct;
                if (newb) {
                    cur_ct = w.ct;
                    ++bu;
                }
                const uint32_t acc = tiles & 1;  // double-buffered accumulator
                mb_wait(&acc_empty[acc], (tiles >> 1) & 1);
                tc_after();
                const uint32_t dacc = tbase + acc * kFN;
#pragma unroll
                for (int s = 0; s < NST; ++s, ++u) {
                    if (newb) mb_wait(&b_full[s], (bu - 1) & 1);
                    const uint32_t sl = u % kFRing;
                    mb_wait(&a_full[sl], (u / kFRing) & 1);
                    {
                        uint64_t da = da0[0];
#pragma unroll
                        for (int i = 1; i < kFRing; ++i)
                            if (sl == static_cast<uint32_t>(i)) da = da0[i];
#pragma unroll
                        for (int j = 0; j < kFKS / 64; ++j)  // the tile's first MMA overwrites the accumulator
                            f4_mma(dacc, da + 16 * j, db0[s] + 16 * j, sfa, sfb, (s | j) != 0);
                    }
                    f4_commit(&a_empty[sl]);  // A stage free once these MMAs are done
                    f4_commit(&b_empty[s]);   // B stage s free once the tile's MMAs on it are done
                }
                f4_commit(&acc_full[acc]);
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue ----------------
        // warp: TMEM lane quarter q (rows 32q..32q+31), 32-column groups h, h + EPW, ... of the tile
        const int q = warp & 3, h = (warp - 4) >> 2;
        const uint32_t tq = tbase + (static_cast<uint32_t>(q * 32) << 16);
        if (h == 0) {  // scale factors: every byte 0x7F = 2^0
            const uint32_t v = 0x7F7F7F7Fu;
            for (int c = 0; c < 64; c += 8)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(tq + kFSfCol + c),
                             "r"(v));
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        tc_before();
        __syncwarp();
        if (lane == 0) {
            mb_arrive(&acc_empty[0]);
            mb_arrive(&acc_empty[1]);
        }
        uint32_t tiles = 0;
        for (int64_t qi = 0;; ++qi) {
            const int slot = static_cast<int>(qi % kFQ);
            mb_wait(&q_full[slot], static_cast<uint32_t>((qi / kFQ) & 1));
            const int64_t ch = q_chunk[slot];
            __syncwarp();
            if (lane == 0) mb_arrive(&q_empty[slot]);
            if (ch < 0) break;
            for (F4Walk w(ch, nrt, T, chunk); w.n > 0; --w.n, w.next(nrt), ++tiles) {
                const uint32_t acc = tiles & 1;
                mb_wait(&acc_full[acc], (tiles >> 1) & 1);
                tc_after();
                // 32 columns at a time, then release the buffer
                constexpr int kG = (kFHW + EPW - 1) / EPW;
                uint32_t par[kG];
#pragma unroll
                for (int c = 0; c < kG; ++c) {
                    par[c] = 0;
                    const int g = h + c * EPW;
                    if (g >= kFHW) break;
                    uint32_t v[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(tq + acc * kFN + 32 * g));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    // exact counts <= 1024: adding 2^23 puts the count's parity in bit 0
                    uint32_t x = 0;
#pragma unroll
                    for (int i = 0; i < 32; ++i) x = __funnelshift_r(x, __float_as_uint(__uint_as_float(v[i]) + 8388608.0f), 1);
                    par[c] = x;
                }
                tc_before();
                __syncwarp();
                if (lane == 0) mb_arrive(&acc_empty[acc]);  // the MMAs of tile + 2 may overwrite it now
                const int64_t row = static_cast<int64_t>(w.rt) * kFM + q * 32 + lane;
                if (row < rows) {
                    // fire-and-forget XOR at L2 (RED): the epilogue never waits on C
                    unsigned* cr = reinterpret_cast<unsigned*>(jb.C.w + (jb.c_r0 + d + row) * jb.C.stride + cw0);
#pragma unroll
                    for (int c = 0; c < kG; ++c) {
                        const int64_t x = static_cast<int64_t>(w.ct) * kFHW + h + c * EPW;  // half-word in the range
                        if (h + c * EPW < kFHW && x < nhw && par[c]) atomicXor(cr + x, par[c]);
                    }
                }
            }
        }
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
    if (tl && tid == 0) atomicMax(tl + 128, gtimer());
}

size_t schur_f4_a_bytes(int64_t rows) { return static_cast<size_t>((rows + kFM - 1) / kFM) * kFMaxStages * kFAStage; }
size_t schur_f4_b_bytes(int64_t words) {
    return static_cast<size_t>((2 * words + kFHW - 1) / kFHW) * kFMaxStages * kFBStage;
}

bool g_pdl = true;  // kernels.cuh: launch_pdl (Tuning::pdl)

// K is always padded to kFMaxStages stages (zero nibbles): the B ring then spans exactly
// one tile, which the loader's B-reload waits rely on (one mbarrier phase per tile)
void launch_schur_f4_expand_a(cudaStream_t s, const F4Job& jb, uint8_t* Ax, int nsm) {
    launch_pdl(k_f4_expand_a, dim3(nsm * 8), dim3(256), 0, s, jb, Ax, kFMaxStages);
}

void launch_schur_f4(cudaStream_t s, const F4Job& jb, const uint8_t* Ax, uint8_t* Bx, unsigned* claim, int nsm,
                     unsigned long long* tl) {
    if (jb.cw1 <= jb.cw0) return;
    launch_pdl(k_f4_expand_b, dim3(nsm * 8), dim3(256), 0, s, jb, Bx, kFMaxStages, claim);
    // 6-deep A ring, 16 epilogue warps (4-deep and 4 tiles per epilogue warp measured slower)
    launch_pdl(k_schur_f4<6, 1>, dim3(nsm), dim3(f4_threads(1)), f4_smem(6), s, jb, Ax, static_cast<const uint8_t*>(Bx),
               claim, tl);
}

void setup_schur_f4_kernels() {
    cudaFuncSetAttribute(k_schur_f4<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(f4_smem(6)));
}

}  // namespace f2g
