// Table-apply / M4RM kernel: C ^= A * B over GF(2).
//
// This one kernel is both
//   * the MMPF table-apply (add_rows_from_table, proj/src/m4ri.cpp:28-38, fed by
//     make_table1, proj/src/mmpf.cpp:54-77) when K is one 64-bit leaf word: every
//     trailing row adds, per 8 coefficient bits, one row of a 256-entry Gray table
//     of pivot-row combinations; and
//   * the Schur-complement multiply of the blocked PLS (addmul_impl,
//     proj/src/mul.cpp:21-68) when K is a whole panel.
// The coefficient bits are read LSB-first (bits_lsb, mul.cpp:61-66): raw bit j of a
// row's coefficient words selects B row map(j).  In the PLS engine the coefficient
// words are the packed L columns themselves (raw pivot columns; a non-pivot column
// is zero in every row the kernel touches and maps to no B row), so no compaction
// pass exists and the L bits are never rewritten.
//
// CTA tile: 1024 rows x 1024 bits of C (16 warps), accumulated in registers over
// all of K.  Per 8-bit chunk of K the CTA builds a 256 x 1024-bit table in SMEM
// (double buffered, 32 KB each) from 8 B rows staged by cp.async three chunks
// ahead; every row then does one 16-byte LDS per thread (8 lanes cover one
// 128-byte table row, so each quarter-warp reads one whole row: conflict-free).
// The coefficient words of the tile's rows are staged in SMEM one K-word ahead.
// SMEM bandwidth bounds it: per chunk 1024 lookups x 128 B + 256 table rows x 128 B.
#include <cstdint>
#include <cstdlib>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kRPT = 16;                         // rows per thread
constexpr int kTNW = 16;                         // 64-bit words per tile row (1024 bits)
constexpr int kTM = kWarps * 4 * kRPT;           // 1024 rows per CTA (4 rows per warp instruction)
#ifndef F2_SCHUR_SINGLE
#define F2_SCHUR_PAIRS 1
#endif
#ifdef F2_SCHUR_PAIRS
constexpr int kStages = 8;                       // B-row ring depth (chunks)
constexpr int kTabs = 4;                         // table buffers: two chunks built while two are read
#else
constexpr int kStages = 4;
constexpr int kTabs = 2;
#endif
constexpr int kMaxMap = kMaxPanelBits;           // K bits held in the SMEM row map
#ifndef F2_BUILD_WARPS
#define F2_BUILD_WARPS 4
#endif
constexpr int kBuildWarps = F2_BUILD_WARPS;      // warps building each chunk's table (4, 8 or 16)

// shared memory carve-up (bytes)
constexpr size_t kOffT = 0;                                   // [kTabs][256][kTNW] u64
constexpr size_t kOffRing = kOffT + kTabs * 256 * kTNW * 8;    // [kStages][8][kTNW]
constexpr size_t kOffA = kOffRing + kStages * 8 * kTNW * 8;    // [2][kTM][2] u64       32 KB (K-word pairs)
constexpr size_t kOffMap = kOffA + 2 * kTM * 8 * 2;            // [kMaxMap] i32         8 KB
constexpr size_t kOffLive = kOffMap + kMaxMap * 4;             // [kMaxMap/8/32] u32
constexpr size_t kSmem = kOffLive + (kMaxMap / 8 / 32) * 4;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(void* p, uint4 v) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) k_table_apply(TableApply p) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* Tb = reinterpret_cast<uint64_t*>(smem + kOffT);
    uint64_t* ring = reinterpret_cast<uint64_t*>(smem + kOffRing);
    uint64_t* abuf = reinterpret_cast<uint64_t*>(smem + kOffA);
    int32_t* bmap = reinterpret_cast<int32_t*>(smem + kOffMap);
    uint32_t* livebits = reinterpret_cast<uint32_t*>(smem + kOffLive);

    int64_t c_r0 = p.c_r0, a_r0 = p.a_r0;
    if (p.row_mode == ROWS_AFTER_LEAF) {
        if (p.st->leaf_kb == 0) return;
        c_r0 = a_r0 = p.st->leaf_r + p.st->leaf_kb;
    } else if (p.row_mode == ROWS_AFTER_PANEL) {
        const int64_t pr = p.rk ? p.rk[0] : p.st->panel_r, pk = p.rk ? p.rk[1] : p.st->panel_kb;
        if (pk == 0) return;
        c_r0 = a_r0 = pr + pk;
    }
    const int64_t row_base = c_r0 + (p.row_tile0 + static_cast<int64_t>(blockIdx.y)) * kTM;
#ifdef F2_TIMELINE
    const int tl_slot = p.st ? static_cast<int>((p.aw0 / 16) & 127) : -1;  // panel index (W = 1024)
    if (tl_slot >= 0 && threadIdx.x == 0 && p.cw1 - p.cw0 > 16) atomicMin(&const_cast<PlsState*>(p.st)->tl[2][tl_slot], gtimer());
#endif
    if (row_base >= p.c_r1) return;
    // K split (gridDim.z > 1): this CTA takes coefficient words [kw0, kw0 + kwn) and
    // XORs its partial product into C atomically (GF(2) addition is order-free)
    const int wps = (p.kw + static_cast<int>(gridDim.z) - 1) / static_cast<int>(gridDim.z);
    const int kw0 = static_cast<int>(blockIdx.z) * wps;
    if (kw0 >= p.kw) return;
    const int kwn = p.kw - kw0 < wps ? p.kw - kw0 : wps;
    const int64_t kbits_l = p.kbits - 64 * kw0 < 64 * kwn ? p.kbits - 64 * kw0 : 64 * kwn;
    if (kbits_l <= 0) return;
    const int64_t aw0_l = p.aw0 + kw0;
    const int64_t* brow_l = p.brow ? p.brow + 64 * kw0 : nullptr;
    const int64_t b_r0_l = p.b_r0 + 64 * kw0;
    const bool split = gridDim.z > 1;
    const int64_t tile_w0 = p.cw0 + static_cast<int64_t>(blockIdx.x) * kTNW;
    const int64_t arow_base = a_r0 + (row_base - c_r0);
    const int64_t nrows = p.c_r1 - row_base < kTM ? p.c_r1 - row_base : kTM;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rq = lane >> 3, wp = lane & 7;
    const int64_t cwa = tile_w0 + 2 * wp, cwb = cwa + 1;
    const bool va = cwa < p.cw1, vb = cwb < p.cw1;
    const int nch = static_cast<int>((kbits_l + 7) / 8);
    const bool mapped = brow_l != nullptr;

    // B row map and live-chunk mask for the whole K range
    if (mapped) {
        for (int j = tid; j < nch * 8; j += kThreads) {
            int64_t r = j < kbits_l ? brow_l[j] : -1;
            bmap[j] = static_cast<int32_t>(r);
        }
        __syncthreads();
        for (int w = tid; w < (nch + 31) / 32; w += kThreads) {
            uint32_t bits = 0;
            for (int b = 0; b < 32 && w * 32 + b < nch; ++b) {
                const int c = w * 32 + b;
                bool any = false;
                for (int k = 0; k < 8; ++k) any |= bmap[c * 8 + k] >= 0;
                bits |= static_cast<uint32_t>(any) << b;
            }
            livebits[w] = bits;
        }
    }

    auto brow_of = [&](int j) -> int64_t {
        if (mapped) return bmap[j];
        return j < kbits_l ? b_r0_l + j : -1;
    };
    auto live = [&](int c) -> bool { return mapped ? ((livebits[c >> 5] >> (c & 31)) & 1u) : c < nch; };

    // B rows of chunk c -> ring stage c % kStages (threads 0..63, one word each)
    // (threads 256..383: warps that never build in the paired schedule)
    auto issue_b = [&](int c) {
        const int tb0 = kThreads - 2 * 8 * kTNW;
        if (tid >= tb0 && tid < tb0 + 8 * kTNW) {
            const int b = (tid - tb0) >> 4, k = (tid - tb0) & 15;
            const int64_t br = brow_of(c * 8 + b);
            const int64_t wcol = tile_w0 + k;
            const bool ok = br >= 0 && wcol < p.cw1;
            const uint64_t* src = ok ? p.B.w + br * p.B.stride + (p.bw0 + (wcol - p.cw0)) : p.B.w;
            cp_async8(ring + ((c % kStages) * 8 + b) * kTNW + k, src, ok);
        }
    };
    // coefficient words 2gg, 2gg+1 of every row of the tile -> abuf[gg & 1][row][0..1]:
    // one 16-byte copy per row (the rows are a stride apart, so every copy is its own
    // global sector either way; pairs halve the copies)
    auto issue_a2 = [&](int gg) {
        const bool al = (aw0_l & 1) == 0;
        const int rem = kwn - 2 * gg;  // valid words in this pair (>= 1)
        for (int r = tid; r < kTM; r += kThreads) {
            const bool ok = r < nrows;
            uint64_t* dst = abuf + ((gg & 1) * kTM + r) * 2;
            const uint64_t* src = p.A.w + (arow_base + r) * p.A.stride + aw0_l + 2 * gg;
            if (al) {
                cp_async16(dst, ok ? src : p.A.w, ok ? (rem >= 2 ? 16 : 8) : 0);
            } else {
                cp_async8(dst, ok ? src : p.A.w, ok);
                cp_async8(dst + 1, ok && rem >= 2 ? src + 1 : p.A.w, ok && rem >= 2);
            }
        }
    };
    // coefficient word g of every row of the tile -> abuf[g & 1]
    auto issue_a = [&](int g) {
        for (int r = tid; r < kTM; r += kThreads) {
            const bool ok = r < nrows;
            const uint64_t* src = ok ? p.A.w + (arow_base + r) * p.A.stride + aw0_l + g : p.A.w;
            cp_async8(abuf + (g & 1) * kTM + r, src, ok);
        }
    };
    // 256-entry table of chunk c: entry e = xor of B rows b with bit b of e (LSB first)
    // built by warps 0..3 only (fewer ring reads): thread = (16-byte column chunk wp,
    // low nibble el of the entry); the high nibble is walked in Gray order
    auto build = [&](int c) {
#ifdef F2_EXP_NOBUILD
        return;
#endif
        if (warp >= kBuildWarps) return;
        const uint64_t* rs = ring + (c % kStages) * 8 * kTNW + 2 * wp;
        const int el = (tid >> 3) & 15;                    // low nibble of the entry
        constexpr int kSeg = 16 / (kBuildWarps / 4);       // Gray steps per thread
        const int k0 = (tid >> 7) * kSeg;                  // first step of this thread's segment
        uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint4 v = lds128(rs + b * kTNW);
            if ((el >> b) & 1) x = xor4(x, v);
        }
        uint4 hv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) hv[b] = lds128(rs + (4 + b) * kTNW);
        const int g0 = k0 ^ (k0 >> 1);
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if ((g0 >> b) & 1) x = xor4(x, hv[b]);
        uint64_t* tb = Tb + (c & 1) * 256 * kTNW + 2 * wp;
#pragma unroll
        for (int s = 0; s < kSeg; ++s) {
            const int k = k0 + s;
            if (s) {
                const int b = __ffs(k) - 1;  // the Gray step k-1 -> k flips bit ctz(k)
                x = xor4(x, b == 0 ? hv[0] : b == 1 ? hv[1] : b == 2 ? hv[2] : hv[3]);
            }
            const int eh = k ^ (k >> 1);
            sts128(tb + (eh * 16 + el) * kTNW, x);
        }
    };

    uint64_t acc0[kRPT], acc1[kRPT];
#pragma unroll
    for (int i = 0; i < kRPT; ++i) {
        const int64_t row = row_base + warp * 64 + rq + 4 * i;
        const bool rv = row < p.c_r1;
        const uint64_t* cr = p.C.w + row * p.C.stride;
        acc0[i] = (rv && va && !split) ? cr[cwa] : 0ull;
        acc1[i] = (rv && vb && !split) ? cr[cwb] : 0ull;
    }

#ifdef F2_SCHUR_PAIRS
    // Two chunks per barrier: while every warp reads tables c, c+1, warps 0-3 build
    // table c+2 and warps 4-7 table c+3, so there is one CTA barrier per 16
    // coefficient bits and each builder warp builds one table per two chunks read.
    // table c by warps 4*grp .. 4*grp+3: thread = (16-byte column chunk wp, low nibble
    // el of the entry); the high nibble walked in Gray order (16 steps)
    auto build_half = [&](int c, int grp) {
        if ((warp >> 2) != grp || c >= nch || !live(c)) return;
        const uint64_t* rs = ring + (c % kStages) * 8 * kTNW + 2 * wp;
        const int el = (tid >> 3) & 15;
        uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint4 v = lds128(rs + b * kTNW);
            if ((el >> b) & 1) x = xor4(x, v);
        }
        uint4 hv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) hv[b] = lds128(rs + (4 + b) * kTNW);
        uint64_t* tb = Tb + (c % kTabs) * 256 * kTNW + 2 * wp;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (k) x = xor4(x, hv[(k & 1) ? 0 : ((k & 2) ? 1 : ((k & 4) ? 2 : 3))]);
            const int eh = k ^ (k >> 1);
            sts128(tb + (eh * 16 + el) * kTNW, x);
        }
    };
    auto lookups = [&](int c, const uint32_t (&aw)[kRPT]) {
        if (c >= nch || !live(c)) return;
        const uint64_t* tb = Tb + (c % kTabs) * 256 * kTNW + 2 * wp;
        const int sh = 8 * (c & 3);
#pragma unroll
        for (int i = 0; i < kRPT; ++i) {
            const unsigned idx = (aw[i] >> sh) & 0xffu;
            const uint4 t = lds128(tb + idx * kTNW);
            acc0[i] ^= static_cast<uint64_t>(t.x) | (static_cast<uint64_t>(t.y) << 32);
            acc1[i] ^= static_cast<uint64_t>(t.z) | (static_cast<uint64_t>(t.w) << 32);
        }
    };
    issue_a2(0);
    for (int c = 0; c < 6; c += 2) {  // chunks 0-1, 2-3, 4-5: one group each
        if (c < nch) issue_b(c);
        if (c + 1 < nch) issue_b(c + 1);
        cp_async_commit();
    }
    cp_async_wait<2>();
    __syncthreads();
    build_half(0, 0);
    build_half(1, 1);
    uint32_t aw[kRPT];
    const int npairs = (nch + 1) / 2;
    for (int pi = 0; pi < npairs; ++pi) {
        const int c = 2 * pi;
        cp_async_wait<1>();
        __syncthreads();
        if ((c & 3) == 0) {  // coefficient bits of chunks c .. c+3
            const int gg = c >> 4;
            const uint32_t* ab = reinterpret_cast<const uint32_t*>(abuf + ((gg & 1) * kTM + warp * 64 + rq) * 2) +
                                 ((c >> 3) & 1) * 2 + ((c >> 2) & 1);
#pragma unroll
            for (int i = 0; i < kRPT; ++i) aw[i] = ab[16 * i];
        }
        build_half(c + 2, 0);
        build_half(c + 3, 1);
        if (c + 6 < nch) issue_b(c + 6);
        if (c + 7 < nch) issue_b(c + 7);
        if ((c & 15) == 0 && 2 * ((c >> 4) + 1) < kwn && 2 * ((c >> 4) + 1) < (nch + 7) / 8) issue_a2((c >> 4) + 1);
        cp_async_commit();
#ifndef F2_EXP_NOLOOKUP
        lookups(c, aw);
        lookups(c + 1, aw);
#endif
    }
#else
    issue_a(0);
    for (int c = 0; c < 3; ++c) {
        if (c < nch) issue_b(c);
        cp_async_commit();
    }
    cp_async_wait<2>();
    __syncthreads();
    if (nch > 0 && live(0)) build(0);

    uint32_t aw[kRPT];  // coefficient bits of the current half K-word (4 chunks)
    const int ngroups = (nch + 7) / 8;
    for (int g = 0; g < ngroups; ++g) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = g * 8 + j;
            if (c < nch) {
                if (c + 3 < nch) issue_b(c + 3);
                if (j == 0 && g + 1 < kwn && g + 1 < ngroups) issue_a(g + 1);
                cp_async_commit();
                cp_async_wait<2>();
                __syncthreads();
                if (j == 0 || j == 4) {
                    const uint32_t* ab = reinterpret_cast<const uint32_t*>(abuf + (g & 1) * kTM + warp * 64 + rq) + (j >> 2);
#pragma unroll
                    for (int i = 0; i < kRPT; ++i) aw[i] = ab[8 * i];
                }
                if (c + 1 < nch && live(c + 1)) build(c + 1);
#ifdef F2_EXP_NOLOOKUP
                if (false) {
#else
                if (live(c)) {
#endif
                    const uint64_t* tb = Tb + (c & 1) * 256 * kTNW + 2 * wp;
#pragma unroll
                    for (int i = 0; i < kRPT; ++i) {
                        const unsigned idx = (aw[i] >> (8 * (j & 3))) & 0xffu;
                        const uint4 t = lds128(tb + idx * kTNW);
                        acc0[i] ^= static_cast<uint64_t>(t.x) | (static_cast<uint64_t>(t.y) << 32);
                        acc1[i] ^= static_cast<uint64_t>(t.z) | (static_cast<uint64_t>(t.w) << 32);
                    }
                }
            }
        }
    }
#endif
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < kRPT; ++i) {
        const int64_t row = row_base + warp * 64 + rq + 4 * i;
        if (row < p.c_r1) {
            uint64_t* cr = p.C.w + row * p.C.stride;
            if (split) {
                if (va) atomicXor(reinterpret_cast<unsigned long long*>(cr + cwa), acc0[i]);
                if (vb) atomicXor(reinterpret_cast<unsigned long long*>(cr + cwb), acc1[i]);
            } else {
                if (va) cr[cwa] = acc0[i];
                if (vb) cr[cwb] = acc1[i];
            }
        }
    }
#ifdef F2_TIMELINE
    if (tl_slot >= 0 && threadIdx.x == 0 && p.cw1 - p.cw0 > 16) atomicMax(&const_cast<PlsState*>(p.st)->tl[3][tl_slot], gtimer());
#endif
}

static size_t table_apply_smem() { return kSmem; }

// One launch over all row tiles, or -- when the tile count leaves a partial last wave
// -- the rows that fill whole waves first, then the remaining row tiles with K split
// across gridDim.z CTAs (atomic XOR into C) so the tail wave is short.  expect_rows
// (the caller's estimate of the device-side row count; <= 0: unknown) only steers
// the split; correctness never depends on it.
void launch_table_apply(cudaStream_t s, const TableApply& t, int nsm, int64_t expect_rows) {
    if (t.cw1 <= t.cw0 || t.kbits <= 0) return;
    if (t.kw == 1) {  // K <= 64: HBM-streaming MMPF kernel
        launch_mmpf_apply(s, t, nsm);
        return;
    }
    const int64_t lo = t.row_mode == ROWS_STATIC ? t.c_r0 : 0;
    const int64_t rows = t.c_r1 - lo;
    if (rows <= 0) return;
    const int64_t nct = (t.cw1 - t.cw0 + kTNW - 1) / kTNW;
    const int64_t nrt = (rows + kTM - 1) / kTM;
    int64_t y0 = nrt;
    int splitk = 1;
    if (expect_rows > 0 && nsm > 0 && t.kw >= 2) {
        const int64_t ert = (expect_rows + kTM - 1) / kTM;  // expected row tiles
        const int64_t tiles = ert * nct;
        const int64_t full_waves = tiles / nsm;
        const int64_t ya = full_waves * nsm / nct;  // row tiles that fit whole waves
        const int64_t tail = (ert - ya) * nct;
        if (ya < ert && tail > 0) {
            int sk = static_cast<int>(nsm / tail);
            if (sk > t.kw) sk = t.kw;
            if (sk >= 2) {
                y0 = ya;
                splitk = sk;
            }
        }
    }
    if (y0 > 0) {
        TableApply a = t;
        a.row_tile0 = 0;
        k_table_apply<<<dim3(static_cast<unsigned>(nct), static_cast<unsigned>(y0 - a.row_tile0), 1), kThreads,
                        table_apply_smem(), s>>>(a);
    }
    if (y0 < nrt) {
        TableApply b = t;
        b.row_tile0 = y0;
        k_table_apply<<<dim3(static_cast<unsigned>(nct), static_cast<unsigned>(nrt - y0), static_cast<unsigned>(splitk)),
                        kThreads, table_apply_smem(), s>>>(b);
    }
}

void setup_m4rm_kernels() {
    cudaFuncSetAttribute(k_table_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(table_apply_smem()));
}

}  // namespace f2g
