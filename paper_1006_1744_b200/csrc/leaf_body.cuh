// Device bodies of the leaf step, shared by the standalone kernels (leaf.cu) and
// the persistent panel kernel (panel.cu).  See leaf.cu for the algorithm.
#pragma once
#include <cstdint>

#include "f2gpu.cuh"

namespace f2g {

namespace {

constexpr unsigned FULL = 0xffffffffu;

constexpr unsigned long long KEY_NONE = ~0ull;

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
    uint32_t lo = __reduce_or_sync(FULL, static_cast<uint32_t>(v));
    uint32_t hi = __reduce_or_sync(FULL, static_cast<uint32_t>(v >> 32));
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// 64-bit minimum as two hardware 32-bit reductions: the high words, then the low words of
// the lanes holding the smallest high word
__device__ __forceinline__ unsigned long long warp_min64(unsigned long long v) {
    const unsigned hi = static_cast<unsigned>(v >> 32);
    const unsigned mh = __reduce_min_sync(FULL, hi);
    const unsigned ml = __reduce_min_sync(FULL, hi == mh ? static_cast<unsigned>(v) : ~0u);
    return (static_cast<unsigned long long>(mh) << 32) | ml;
}

// mask of bits strictly above bit c (c in 0..63)
__device__ __forceinline__ uint64_t above(int c) { return c >= 63 ? 0ull : (~0ull << (c + 1)); }

__device__ __forceinline__ int omap_hash(int64_t p) {
    return static_cast<int>((static_cast<uint64_t>(p) * 0x9E3779B97F4A7C15ull) >> 57);  // 7 bits
}

struct Omap {
    int64_t key[kOmapSlots];
    int64_t val[kOmapSlots];
};

__device__ __forceinline__ int64_t omap_get(const Omap& om, int64_t p) {
    int h = omap_hash(p);
    for (int i = 0; i < kOmapSlots; ++i) {
        int s = (h + i) & (kOmapSlots - 1);
        int64_t k = om.key[s];
        if (k == p) return om.val[s];
        if (k < 0) return p;
    }
    return p;
}

__device__ __forceinline__ void omap_put(Omap& om, int64_t p, int64_t v) {
    int h = omap_hash(p);
    for (int i = 0; i < kOmapSlots; ++i) {
        int s = (h + i) & (kOmapSlots - 1);
        if (om.key[s] == p || om.key[s] < 0) {
            om.key[s] = p;
            om.val[s] = v;
            return;
        }
    }
}

template <int S>
__device__ __forceinline__ uint64_t pick(const uint64_t (&v)[S], int s) {
    uint64_t r = v[0];
#pragma unroll
    for (int i = 1; i < S; ++i)
        if (s == i) r = v[i];
    return r;
}

template <int S>
__device__ __forceinline__ int32_t pick(const int32_t (&v)[S], int s) {
    int32_t r = v[0];
#pragma unroll
    for (int i = 1; i < S; ++i)
        if (s == i) r = v[i];
    return r;
}

}  // namespace


// ---- dense fast path ---------------------------------------------------------------
// The first 128 positions of the current order ("the window") are transposed into
// column form: column c of the leaf is a 128-bit mask over the window's slots.
// Warp 0 runs the Gaussian pivot rule on the masks, lane l owning columns l and l+32:
// per column, candidates = its bits at slots >= t; the lowest is the pivot (the first
// row in the current order, exactly gauss.cpp:33-40, because the window is a prefix
// of that order); its slot swaps with slot t (a two-bit swap in every mask, :44);
// rows below with a 1 receive the pivot row from the next column on (one masked XOR
// per column, :47-49).  A column without candidates is decided only when no rows lie
// past the window; otherwise the leaf falls back to the general search below
// (rank-deficient / sparse inputs).
//
// The panel kernel (panel.cu, pipe_fast_leaf) drives these warps on its carried
// 128-row window and then solves the pivot rows over the rest of the panel.
struct U128 {
    uint64_t lo, hi;
};

// (nlo, nhi) = -(lo, hi) as one 128-bit two's complement (one carry chain)
__device__ __forceinline__ void neg128(uint64_t lo, uint64_t hi, uint64_t& nlo, uint64_t& nhi) {
    asm("sub.cc.u64 %0, 0, %2;\n\tsubc.u64 %1, 0, %3;\n" : "=l"(nlo), "=l"(nhi) : "l"(lo), "l"(hi));
}

__device__ __forceinline__ uint32_t warp_transpose32(uint32_t v, int lane) {
    // lane i holds bits (i, 0..31) -> lane j holds bits (0..31, j)
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1, m ^= m << j) {
        const uint32_t x = __shfl_xor_sync(FULL, v, j);
        const bool up = lane & j;
        const uint32_t lo = up ? x : v, hi = up ? v : x;
        const uint32_t t = ((lo >> j) ^ hi) & m;
        v ^= up ? t : (t << j);
    }
    return v;
}

struct FastSmem {
    uint32_t colw[64 * 4];       // leaf columns: 4 x 32 slots each
    uint64_t linv[64];           // rows of L11^{-1} over pivot indices
    uint64_t rraw[64];           // the same rows in raw leaf-column coordinates
    int posc[64];                // leaf column -> pivot index, -1
    int64_t phys[128];           // pre-leaf physical row of each slot
    int step_p[64], step_c[64];  // pivot steps
    int src[128];                // slot s now holds the pre-leaf content of slot src[s]
    uint64_t uf[64];             // pivot rows' final leaf words
    int wcount[4];
    int final_kb;                // -1: fell back
    // two-warp search: published steps (the selecting warp writes, the other replays)
    ulonglong2 step_m[64];       // step t's candidate mask: the pivot column's bits at slots >= t
    uint32_t ufl[64], ufh[64];   // pivot rows' leaf words, columns 0-31 / 32-63
    uint64_t fbas[64];           // finalize basis
    uint64_t cfin[64];           // post-search column masks, slots 0..63 (bit l = row l's bit in column c)
    uint32_t ainv[32], brows[32];
    volatile int q_n;            // published progress: (columns processed << 8) | steps
#ifdef F2_LEAF_CLOCKS
    long long clk[2][2];         // selecting loop start / end per phase
#endif
};

// Warp 0: the column-form pivot rule on F.colw (leaf columns as 128-slot masks).
// Fills step_p/step_c, final_kb (-1: a column needs rows past the window), the pivot
// rows' final leaf words uf and, with want_linv, the rows of L11^{-1}.
__device__ __forceinline__ void warp0_pivots(FastSmem& F, int lw, bool more, bool want_linv, PlsState* st) {
    const int lane = threadIdx.x & 31;
        U128 C0, C1;
        C0.lo = F.colw[lane * 4] | (static_cast<uint64_t>(F.colw[lane * 4 + 1]) << 32);
        C0.hi = F.colw[lane * 4 + 2] | (static_cast<uint64_t>(F.colw[lane * 4 + 3]) << 32);
        C1.lo = F.colw[(lane + 32) * 4] | (static_cast<uint64_t>(F.colw[(lane + 32) * 4 + 1]) << 32);
        C1.hi = F.colw[(lane + 32) * 4 + 2] | (static_cast<uint64_t>(F.colw[(lane + 32) * 4 + 3]) << 32);
                int t = 0;
        bool ok = true;
        for (int c = 0; c < lw; ++c) {
            const uint64_t srclo = c < 32 ? C0.lo : C1.lo, srchi = c < 32 ? C0.hi : C1.hi;
            const uint64_t mlo = __shfl_sync(FULL, srclo, c & 31);
            const uint64_t mhi = __shfl_sync(FULL, srchi, c & 31);
            const uint64_t clo = mlo & (~0ull << t);  // t <= 63 here
            if ((clo | mhi) == 0) {
                if (more) {
                    ok = false;
                    break;
                }
                continue;  // zero column among all remaining rows: no pivot (gauss.cpp:36-41)
            }
            const int p = clo ? __ffsll(static_cast<long long>(clo)) - 1 : 63 + __ffsll(static_cast<long long>(mhi));
            const uint64_t tb = 1ull << t;
            const uint64_t plo = p < 64 ? (1ull << p) : 0ull, phi = p < 64 ? 0ull : (1ull << (p - 64));
            // swap slots t and p in every mask (a no-op when p == t)
            {
                const uint64_t d0 = (((C0.lo & tb) != 0) != (((C0.lo & plo) | (C0.hi & phi)) != 0)) ? ~0ull : 0ull;
                C0.lo ^= d0 & (tb | plo);
                C0.hi ^= d0 & phi;
                const uint64_t d1 = (((C1.lo & tb) != 0) != (((C1.lo & plo) | (C1.hi & phi)) != 0)) ? ~0ull : 0ull;
                C1.lo ^= d1 & (tb | plo);
                C1.hi ^= d1 & phi;
            }
            // column c after the swap: bit t set, bit p cleared; rows below t with a 1
            const uint64_t elo = (mlo & ~plo) & (t == 63 ? 0ull : (~0ull << (t + 1)));
            const uint64_t ehi = mhi & ~phi;
            const bool a0 = lane > c && (C0.lo & tb);
            const bool a1 = lane + 32 > c && (C1.lo & tb);
            C0.lo ^= a0 ? elo : 0ull;
            C0.hi ^= a0 ? ehi : 0ull;
            C1.lo ^= a1 ? elo : 0ull;
            C1.hi ^= a1 ? ehi : 0ull;
            F.step_p[t] = p;  // same value from every lane: one store
            F.step_c[t] = c;
            ++t;
        }
        F2_STAMP(st, 17);
        if (lane == 0) F.final_kb = ok ? t : -1;
        if (ok) {
            // pivot rows' final leaf words: slots 0..63 of the 64 columns back to row form
            const uint32_t r00 = warp_transpose32(static_cast<uint32_t>(C0.lo), lane);        // slots 0-31, cols 0-31
            const uint32_t r01 = warp_transpose32(static_cast<uint32_t>(C1.lo), lane);        // slots 0-31, cols 32-63
            const uint32_t r10 = warp_transpose32(static_cast<uint32_t>(C0.lo >> 32), lane);  // slots 32-63
            const uint32_t r11 = warp_transpose32(static_cast<uint32_t>(C1.lo >> 32), lane);
            const uint64_t u0 = r00 | (static_cast<uint64_t>(r01) << 32);
            const uint64_t u1 = r10 | (static_cast<uint64_t>(r11) << 32);
            F.uf[lane] = u0;
            F.uf[lane + 32] = u1;
            if (want_linv) {
                // L11^{-1}: row l = e_l + sum over t < l with L bit of l at q_t of row t
                __syncwarp();
                uint64_t R0 = 1ull << lane, R1 = 1ull << (lane + 32);
                for (int tt = 0; tt < t; ++tt) {
                    const int qt = F.step_c[tt];
                    const uint64_t Rt = __shfl_sync(FULL, tt < 32 ? R0 : R1, tt & 31);
                    if (lane > tt && ((u0 >> qt) & 1ull)) R0 ^= Rt;
                    if (lane + 32 > tt && ((u1 >> qt) & 1ull)) R1 ^= Rt;
                }
                F.linv[lane] = R0;
                F.linv[lane + 32] = R1;
            }
        }
    }


// One warp: rows of L11^{-1} over pivot indices from the pivot rows' leaf words:
// row l = e_l + sum over t < l with the L bit of l at column q_t of row t.
__device__ __forceinline__ void warp_linv(FastSmem& F, int kb) {
    const int lane = threadIdx.x & 31;
    const uint64_t u0 = F.uf[lane], u1 = F.uf[lane + 32];
    // the L bits of rows lane and lane+32 gathered into pivot-index order first, so the
    // 64-step chain is one shuffle and two masked XORs per step
    uint64_t c0 = 0, c1 = 0;
    for (int tt = 0; tt < kb; ++tt) {
        const int qt = F.step_c[tt];
        c0 |= ((u0 >> qt) & 1ull) << tt;
        c1 |= ((u1 >> qt) & 1ull) << tt;
    }
    c0 &= lane == 0 ? 0ull : (~0ull >> (64 - lane));  // strictly below the row's own index
    uint64_t R0 = 1ull << lane, R1 = 1ull << (lane + 32);
#pragma unroll 4
    for (int tt = 0; tt < 32; ++tt) {
        const uint64_t Rt = __shfl_sync(FULL, R0, tt);
        R0 ^= ((c0 >> tt) & 1ull) ? Rt : 0ull;
        R1 ^= ((c1 >> tt) & 1ull) ? Rt : 0ull;
    }
    c1 &= lane == 0 ? ~0ull >> 32 : (~0ull >> (32 - lane));  // t < lane + 32
#pragma unroll 4
    for (int tt = 32; tt < 64; ++tt) {
        const uint64_t Rt = __shfl_sync(FULL, R1, tt - 32);
        R1 ^= ((c1 >> tt) & 1ull) ? Rt : 0ull;
    }
    F.linv[lane] = R0;
    F.linv[lane + 32] = R1;
}

// Warps 0 and 1: rows of L11^{-1} (pivot-index coordinates) from the post-search
// column masks.  Column q_t's mask holds, in bit l, row l's bit at that column, so
// one transpose gives every row's L bits in pivot order; then L11 = [A 0; B C] in
// 32x32 blocks: A^{-1} (warp 0) and C^{-1} (warp 1) by 32-step shuffle chains in
// parallel, and the off-diagonal block C^{-1} B A^{-1} by two independent passes.
__device__ __forceinline__ void pair_linv(FastSmem& F, int kb) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int tt = 32 * w + lane;
    const uint64_t vt = tt < kb ? F.cfin[F.step_c[tt]] : 0ull;  // bit l: L[l][tt] (for l > tt)
    uint32_t rows, rowsb = 0;
    if (w == 0) {
        rows = warp_transpose32(static_cast<uint32_t>(vt), lane) & ((1u << lane) - 1u);  // A rows
        rowsb = warp_transpose32(static_cast<uint32_t>(vt >> 32), lane);                 // B rows
    } else {
        (void)warp_transpose32(static_cast<uint32_t>(vt), lane);
        rows = warp_transpose32(static_cast<uint32_t>(vt >> 32), lane) & ((1u << lane) - 1u);  // C rows
    }
    uint32_t R = 1u << lane;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) {
        const uint32_t Rt = __shfl_sync(FULL, R, t);
        R ^= ((rows >> t) & 1u) ? Rt : 0u;
    }
    if (w == 0) {
        F.ainv[lane] = R;
        F.brows[lane] = rowsb;
    }
    asm volatile("bar.sync 2, 64;\n" ::: "memory");
    if (w == 0) {
        F.linv[lane] = R;
    } else {
        const uint32_t b = F.brows[lane];
        uint32_t y = 0;  // (B A^{-1}) row
#pragma unroll 8
        for (int t = 0; t < 32; ++t) y ^= ((b >> t) & 1u) ? F.ainv[t] : 0u;
        uint32_t z = 0;  // (C^{-1} B A^{-1}) row
#pragma unroll 8
        for (int sidx = 0; sidx < 32; ++sidx) {
            const uint32_t ys = __shfl_sync(FULL, y, sidx);
            z ^= ((R >> sidx) & 1u) ? ys : 0u;
        }
        F.linv[32 + lane] = static_cast<uint64_t>(z) | (static_cast<uint64_t>(R) << 32);
    }
}

// Warps 0 and 1: the same pivot rule with the columns split, lane l of warp w owning
// column 32w + l.  Warp 0 selects the pivots of columns 0-31 while warp 1 replays each
// published step (slot swap + masked XOR) on its columns; then warp 1 selects columns
// 32-63 while warp 0 replays the swaps.  Each selecting step touches one column mask
// per lane instead of two.  Same outputs as warp0_pivots.
__device__ __forceinline__ void two_warp_pivots(FastSmem& F, int lw, bool more, bool want_linv) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int col = 32 * w + lane;
    U128 C;
    if (w < 2) {
        C.lo = F.colw[col * 4] | (static_cast<uint64_t>(F.colw[col * 4 + 1]) << 32);
        C.hi = F.colw[col * 4 + 2] | (static_cast<uint64_t>(F.colw[col * 4 + 3]) << 32);
    } else {
        // warp 2 tracks the slot permutation: lane b < 7 holds the mask of slots whose
        // pre-leaf index has bit b set; it replays every swap, so at the end bit b of
        // slot s's source index sits in bit s of mask b
        const uint64_t pat[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                 0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
        C.lo = lane < 6 ? pat[lane] : 0ull;
        C.hi = lane < 6 ? pat[lane] : (lane == 6 ? ~0ull : 0ull);
    }
    if (threadIdx.x == 0) {
        F.q_n = 0;
    }
    asm volatile("bar.sync 1, 96;\n" ::: "memory");
    // step t from its candidate mask m: the pivot is m's lowest bit, the rows to
    // eliminate are m's other bits (all below slot t after the swap)
    auto apply = [&](int t, ulonglong2 m, bool xr) {
        const uint64_t tb = 1ull << t;
        const uint64_t plo = m.x & (0ull - m.x), phi = m.x ? 0ull : (m.y & (0ull - m.y));
        const uint64_t elo = m.x ^ plo, ehi = m.y ^ phi;
        const uint64_t d = (((C.lo & tb) != 0) != (((C.lo & plo) | (C.hi & phi)) != 0)) ? ~0ull : 0ull;
        C.lo ^= d & (tb | plo);
        C.hi ^= d & phi;
        const bool a = xr && (C.lo & tb);
        C.lo ^= a ? elo : 0ull;
        C.hi ^= a ? ehi : 0ull;
    };
    // The selecting warp releases (columns processed << 8) | steps after every column; a
    // replaying warp applies the steps it sees and knows the phase is over when the column
    // count reaches the phase's end (and whether it was decidable from the step count).
    auto progress = [&]() {
        unsigned v;
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(const_cast<int*>(&F.q_n)))) : "memory");
        return v;
    };
    int t = 0;
    bool ok = true;
    if (w == 2) {
        for (int phase = 0; phase < 2 && ok; ++phase) {
            if (32 * phase >= lw) break;
            const int c0 = 32 * phase, c1 = lw < c0 + 32 ? lw : c0 + 32, t0 = t;
            while (true) {
                const unsigned v = progress();
                for (; t < static_cast<int>(v & 255u); ++t) apply(t, F.step_m[t], false);
                if (static_cast<int>(v >> 8) >= c1) {
                    ok = ok && !(more && t - t0 < c1 - c0);
                    break;
                }
            }
        }
        // Written whatever this warp's own `ok` says: the tracker may read the progress word
        // only after the other warp has started publishing phase 1, apply some of those steps
        // before leaving phase 0, and then undercount phase 1 -- its `ok` is not authoritative
        // (warp 0's final_kb is), while its masks, having applied every step in order, are.
        // (Gating this store on the tracker's `ok` once left stale slot sources behind, so a
        // leaf's pivot rows went to the wrong physical rows in rare runs.)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint64_t m = k < 2 ? C.lo : C.hi;
            const uint32_t piece = static_cast<uint32_t>(m >> (32 * (k & 1)));
            F.src[32 * k + lane] = static_cast<int>(warp_transpose32(piece, lane) & 127u);
        }
    } else
    for (int phase = 0; phase < 2; ++phase) {
        const int c0 = 32 * phase, c1 = lw < c0 + 32 ? lw : c0 + 32;
        if (w == phase) {
            // select the pivots of columns c0 .. c1-1.  Branch-free: a column without a
            // pivot is a masked no-op step, so the chain from one shuffle to the next has
            // no convergence points (after a column the window cannot decide the later
            // steps still run, and the leaf is discarded)
            const int t0 = t;
            F2_CLK(if (lane == 0) F.clk[phase][0] = clock64();)
            uint64_t tb = 1ull << t, tm = ~0ull << t;  // slot t, slots >= t
#pragma unroll 2
            for (int c = c0; c < c1; ++c) {
                const uint64_t mlo = __shfl_sync(FULL, C.lo, c & 31);
                const uint64_t mhi = __shfl_sync(FULL, C.hi, c & 31);
                // candidates: slots >= t; the pivot is the lowest (as a bit: x & -x over
                // the 128-bit mask), the rows to eliminate the others.  Every quantity is
                // masked, none branched on, and the pivot's index is left to the readers of
                // the candidate mask.
                const uint64_t clo = mlo & tm;
                uint64_t plo, phi;
                neg128(clo, mhi, plo, phi);
                plo &= clo;
                phi &= mhi;
                const bool zero = (plo | phi) == 0;
                const uint64_t elo = clo ^ plo, ehi = mhi ^ phi;
                const uint64_t tz = zero ? 0ull : tb;
                {  // apply step t to this lane's column (a no-op when zero)
                    const uint64_t d = (((C.lo & tz) != 0) != (((C.lo & plo) | (C.hi & phi)) != 0)) ? ~0ull : 0ull;
                    C.lo ^= d & (tz | plo);
                    C.hi ^= d & phi;
                    const bool a = col > c && (C.lo & tz);
                    C.lo ^= a ? elo : 0ull;
                    C.hi ^= a ? ehi : 0ull;
                }
                // only real steps are stored (predicated, not branched): every lane then
                // writes identical values, so a reader acquiring the count from any lane's
                // release sees the step whichever lane's store it observes
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.u32 p, %0, 0;\n\t"
                    "@p st.shared.v2.u64 [%1], {%2, %3};\n\t"
                    "@p st.shared.u32 [%4], %5;\n\t}"
                    ::"r"(static_cast<unsigned>(!zero)),
                    "r"(static_cast<unsigned>(__cvta_generic_to_shared(&F.step_m[t]))), "l"(clo), "l"(mhi),
                    "r"(static_cast<unsigned>(__cvta_generic_to_shared(&F.step_c[t]))), "r"(c)
                    : "memory");
                t += zero ? 0 : 1;
                tb = zero ? tb : tb << 1;
                tm = zero ? tm : tm << 1;
                // every lane stored the same step and releases the same word: no branch
                asm volatile("st.release.cta.shared.u32 [%0], %1;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(const_cast<int*>(&F.q_n)))), "r"(static_cast<unsigned>(((c + 1) << 8) | t)) : "memory");
            }
            // a column without candidates is undecidable when rows past the window could hold them
            ok = ok && !(more && t - t0 < c1 - c0);  // (c1 < c0 for narrow leaves)
            F2_CLK(if (lane == 0) F.clk[phase][1] = clock64();)
        } else if (c0 < lw) {
            // replay the other warp's steps as they are published
            const int t0 = t;
            while (true) {
                const unsigned v = progress();
                for (; t < static_cast<int>(v & 255u); ++t) apply(t, F.step_m[t], w > phase);
                if (static_cast<int>(v >> 8) >= c1) {
                    ok = ok && !(more && t - t0 < c1 - c0);
                    break;
                }
            }
        }
        if (!ok) break;
    }
    if (lane == 0 && w == 0) F.final_kb = ok ? t : -1;
    if (w < 2) F.cfin[col] = C.lo;
    if (ok && w < 2 && col < t) {  // pivot slot of every step, from its candidate mask
        const ulonglong2 m = F.step_m[col];
        F.step_p[col] = m.x ? __ffsll(static_cast<long long>(m.x)) - 1 : 63 + __ffsll(static_cast<long long>(m.y));
    }
    if (ok && w < 2) {
        // pivot rows' final leaf words (slots 0..63), this warp's 32 columns
        const uint32_t r0 = warp_transpose32(static_cast<uint32_t>(C.lo), lane);
        const uint32_t r1 = warp_transpose32(static_cast<uint32_t>(C.lo >> 32), lane);
        if (w == 0) {
            F.ufl[lane] = r0;
            F.ufl[lane + 32] = r1;
        } else {
            F.ufh[lane] = r0;
            F.ufh[lane + 32] = r1;
        }
    }
    asm volatile("bar.sync 1, 96;\n" ::: "memory");
    if (ok && w == 0) {
        const uint64_t u0 = F.ufl[lane] | (static_cast<uint64_t>(F.ufh[lane]) << 32);
        const uint64_t u1 = F.ufl[lane + 32] | (static_cast<uint64_t>(F.ufh[lane + 32]) << 32);
        F.uf[lane] = u0;
        F.uf[lane + 32] = u1;
        if (want_linv) warp_linv(F, t);
    }
}

// One CTA of 1024 threads.  Warp 0 keeps a sliding window of 32 consecutive
// positions (lane l holds position bb + l), eagerly eliminated, and finds pivots
// there without block-level synchronisation:
//   * fast path: the row at the next pivot position p has a 1 in the next
//     unprocessed column -> it is the pivot, no swap (the common dense case);
//   * otherwise the leftmost nonzero column c* among the window's candidates;
//     exact whenever c* is the next column or nothing lies past the window.
// Once 16 candidates are consumed the window slides to start at p (new rows are
// caught up on the pivots so far).  When rows past the window could hold an
// earlier column, the whole block scans them, catching each row up, for the
// leftmost column below c* (SURVEY.md §7 "Hard parts" 1).
//
// Positions are relative to base = st->r; `src` is the relative (pre-leaf)
// position of the content a lane holds.  Rows are read through pmap.
// The general search of the panel kernel (its fast window could not decide the leaf).
//
// Sparse leaves (a column's candidates scattered over the whole matrix, so nearly every
// column needs a scan): the first scan of the leaf visits every position past the window
// and keeps each row whose caught-up leaf word is nonzero in a compact list in `cmem`
// (cap entries: position, source, word, pivots applied).  A row whose leaf word is zero is
// never touched by the leaf's eliminations and never becomes a candidate, so the later
// scans of the leaf visit the list only (in SMEM, catching each entry up on the new
// pivots), with the same keys -- (column, position) minimum -- as the full scan.  An
// outside pivot's position receives the window row it swaps with; its entry is
// updated in place.  More nonzero rows than cap: full scans, as without a list.
static __device__ __noinline__ void leaf_pivot_body(const Mat& A, int64_t wl, int lw, int first_in_panel, int leaf_in_panel,
                                int panel_bits, PlsState* st, int64_t* P, int64_t* Qp, int64_t* pmap,
                                int64_t qcol_off, uint8_t* cmem = nullptr, int cap = 0) {
    __syncthreads();
    __shared__ uint64_t s_u[64];
    __shared__ uint64_t s_uf[64];
    __shared__ int s_q[64];
    __shared__ Omap s_om;
    __shared__ int64_t s_mv_dst[kMaxSwaps], s_mv_phys[kMaxSwaps];
    __shared__ int s_nmv;
    __shared__ unsigned long long s_red[32];
    __shared__ unsigned long long s_best;
    __shared__ uint64_t s_bword;
    __shared__ int64_t s_bsrc;
    __shared__ int s_cmd, s_col, s_lim, s_t, s_ob;
    __shared__ int s_nom;
    __shared__ int64_t s_om_pos[64];
    __shared__ int s_cn, s_cstate, s_bidx;  // compact list: entries, 0 none yet / 1 valid / 2 off
    uint64_t* const c_w = reinterpret_cast<uint64_t*>(cmem);
    int* const c_pos = reinterpret_cast<int*>(cmem + 8 * static_cast<size_t>(cap));
    int* const c_src = c_pos + cap;
    uint8_t* const c_tt = reinterpret_cast<uint8_t*>(c_src + cap);

#ifdef F2_LEAF_PROFILE
    long long c_start = clock64();
#define F2_MARK(i) do { if (threadIdx.x == 0) st->dbg[i] = clock64() - c_start; } while (0)
#else
#define F2_MARK(i) do { } while (0)
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int64_t m = A.m, stride = A.stride;
    const int64_t base = st->r;
    const int64_t span64 = m - base;
    const int span = span64 > (1 << 30) ? (1 << 30) : static_cast<int>(span64);  // positions left

    for (int i = tid; i < kOmapSlots; i += blockDim.x) s_om.key[i] = -1;
    if (first_in_panel)
        for (int i = tid; i < panel_bits; i += blockDim.x) st->brow[i] = -1;
    if (tid == 0) {
        s_nom = 0;
        if (first_in_panel) st->nmoved = 0;
        s_cn = 0;
        s_cstate = cmem && cap > 0 ? 0 : 2;
        s_bidx = -1;
    }
    __syncthreads();

    uint64_t w = 0;
    int src = 0;
    int t = 0, col = 0, p = 0, bb = 0, nmv = 0;

    // fresh content of relative position x (outside the registers), caught up on tt pivots
    // apply pivots 0..tt-1 to a pre-leaf word (loads independent of the chain)
    auto catch_up = [&](uint64_t v, int tt) -> uint64_t {
        int l = 0;
        for (; l + 4 <= tt; l += 4) {
            const uint64_t u0 = s_u[l], u1 = s_u[l + 1], u2 = s_u[l + 2], u3 = s_u[l + 3];
            const int q0 = s_q[l], q1 = s_q[l + 1], q2 = s_q[l + 2], q3 = s_q[l + 3];
            v ^= ((v >> q0) & 1ull) ? u0 : 0ull;
            v ^= ((v >> q1) & 1ull) ? u1 : 0ull;
            v ^= ((v >> q2) & 1ull) ? u2 : 0ull;
            v ^= ((v >> q3) & 1ull) ? u3 : 0ull;
        }
        for (; l < tt; ++l) v ^= ((v >> s_q[l]) & 1ull) ? s_u[l] : 0ull;
        return v;
    };
    // fresh content of relative position x (outside the registers), caught up on tt pivots
    auto load_fresh = [&](int x, int tt, uint64_t& wo, int& so) {
        if (x >= span) {
            wo = 0;
            so = x;
            return;
        }
        const int64_t sabs = omap_get(s_om, base + x);
        so = static_cast<int>(sabs - base);
        wo = catch_up(ldw(A.w + ldi(pmap + sabs) * stride + wl), tt);
    };
    // raw pre-leaf word of relative position x, loaded early for the next slide
    uint64_t pf_w = 0;
    auto prefetch = [&](int x) { pf_w = x < span ? ldw(A.w + ldi(pmap + base + x) * stride + wl) : 0ull; };

    // append (position base+x <- pre-leaf position base+sx) to the move list, warp-wide
    auto record_moves = [&](bool moved, int x, int sx) {
        const unsigned b = __ballot_sync(FULL, moved);
        if (moved) {
            const int idx = nmv + __popc(b & ((1u << lane) - 1));
            s_mv_dst[idx] = base + x;
            s_mv_phys[idx] = pmap[base + sx];
        }
        nmv += __popc(b);
    };
    auto record_pivot = [&](int cstar, uint64_t u, int64_t pabs_src) {
        if (lane == 0) {
            s_u[t] = u & above(cstar);
            s_uf[t] = u;
            s_q[t] = cstar;
            P[base + p] = pabs_src;
            Qp[base + p] = qcol_off + wl * 64 + cstar;
        }
        __syncwarp();
    };

    F2_MARK(0);
    if (warp == 0) {
        load_fresh(lane, 0, w, src);
        prefetch(32 + lane);
    }
    F2_MARK(1);
    F2_STAMP(st, 10);

    while (true) {
        if (warp == 0) {
            int cmd = 0, lim = 64;
            while (true) {
                if (col >= lw || p >= span) {
                    cmd = 0;
                    break;
                }
                if (p - bb >= 16 && bb + 32 < span) {  // slide the window to start at p
                    __syncwarp();
                    const int d = p - bb;
                    record_moves(lane < d && src != bb + lane, bb + lane, src);
                    uint64_t wn = __shfl_down_sync(FULL, w, d);
                    int sn = __shfl_down_sync(FULL, src, d);
                    const uint64_t pw = __shfl_sync(FULL, pf_w, (lane + d) & 31);
                    if (lane >= 32 - d) {
                        const int x = p + lane;
                        if (s_nom != 0 || x >= span) {
                            load_fresh(x, t, wn, sn);
                        } else {
                            wn = catch_up(pw, t);
                            sn = x;
                        }
                    }
                    w = wn;
                    src = sn;
                    bb = p;
                    prefetch(bb + 32 + lane);
                }
                const int pr = p - bb;
                const bool cand = lane >= pr;
                unsigned hit = __ballot_sync(FULL, cand && ((w >> col) & 1ull));
                int cstar = col;
                if (hit == 0) {
                    const uint64_t any = warp_or64(cand ? (w & (~0ull << col)) : 0ull);
                    cstar = any ? __ffsll(static_cast<long long>(any)) - 1 : 64;
                    if (bb + 32 < span) {  // rows past the window may hold an earlier column
                        cmd = 1;
                        lim = cstar;
                        break;
                    }
                    if (!any) {
                        cmd = 0;
                        break;
                    }
                    hit = __ballot_sync(FULL, cand && ((w >> cstar) & 1ull));
                }
                const int ln = __ffs(hit) - 1;
                const uint64_t u = __shfl_sync(FULL, w, ln);
                if (ln != pr) {
                    const uint64_t wp = __shfl_sync(FULL, w, pr);
                    const int usrc = __shfl_sync(FULL, src, ln);
                    const int psrc = __shfl_sync(FULL, src, pr);
                    if (lane == ln) {
                        w = wp;
                        src = psrc;
                    }
                    if (lane == pr) {
                        w = u;
                        src = usrc;
                    }
                }
                const uint64_t us = u & above(cstar);
                if (lane > pr && ((w >> cstar) & 1ull)) w ^= us;
                if (lane == 0) {
                    s_u[t] = us;
                    s_uf[t] = u;
                    s_q[t] = cstar;
                    P[base + p] = base + bb + ln;
                    Qp[base + p] = qcol_off + wl * 64 + cstar;
                }
#ifdef F2_LEAF_PROFILE
                if (lane == 0 && t < 11) st->dbg[5 + t] = clock64() - c_start;
#endif
                ++t;
                ++p;
                col = cstar + 1;
            }
            __syncwarp();
            if (lane == 0) {
                s_cmd = cmd;
                s_col = col;
                s_lim = lim;
                s_t = t;
                s_ob = bb + 32;
            }
            F2_MARK(2);
        }
        __syncthreads();
        if (s_cmd == 0) break;
        F2_STAMP(st, 14);

        // ---- block-wide scan of positions [ob, m) for the leftmost column in [col, lim)
        const int64_t ob = base + s_ob;
        if (s_cstate == 1) {  // the leaf's nonzero rows past the first scan's window, in SMEM
            // keys as 32 bits (column << 24 | position - ob: the list exists only while the span
            // fits 24 bits), one hardware min-reduction per warp and one across the warps
            const int c0 = s_col, tt = s_t, lim = s_lim, cn = s_cn;
            unsigned key = ~0u;  // this thread's best entry
            uint64_t bv = 0;
            int bi = -1;
            for (int i = tid; i < cn; i += blockDim.x) {
                const int64_t pp = base + c_pos[i];
                if (pp < ob) continue;
                uint64_t v = c_w[i];
                const int ti = c_tt[i];
                if (ti < tt) {
                    for (int l = ti; l < tt; ++l)
                        if ((v >> s_q[l]) & 1ull) v ^= s_u[l];
                    c_w[i] = v;
                    c_tt[i] = static_cast<uint8_t>(tt);
                }
                uint64_t z = v & (~0ull << c0);
                if (lim < 64) z &= (1ull << lim) - 1;
                if (z) {
                    const unsigned kk = (static_cast<unsigned>(__ffsll(static_cast<long long>(z)) - 1) << 24) |
                                        static_cast<unsigned>(pp - ob);
                    if (kk < key) {
                        key = kk;
                        bv = v;
                        bi = i;
                    }
                }
            }
            const unsigned k = __reduce_min_sync(FULL, key);
            if (lane == 0) s_red[warp] = k;
            __syncthreads();
            if (warp == 0) {
                const unsigned kk = __reduce_min_sync(FULL, lane < nwarps ? static_cast<unsigned>(s_red[lane]) : ~0u);
                if (lane == 0)
                    s_best = kk == ~0u ? KEY_NONE
                                       : (static_cast<unsigned long long>(kk >> 24) << 48) | (kk & 0xFFFFFFu);
            }
            __syncthreads();
            if (key != ~0u && key == k && key == static_cast<unsigned>(((s_best >> 48) << 24) | (s_best & 0xFFFFFFu))) {
                s_bword = bv;
                s_bsrc = base + c_src[bi];
                s_bidx = bi;
            }
            __syncthreads();
        } else {
            const int c0 = s_col, tt = s_t;
            int lim = s_lim;
            const bool build = s_cstate == 0;  // first scan: every position, listing the nonzero rows
            if (tid == 0) s_best = KEY_NONE;
            __syncthreads();
            for (int64_t b = ob; b < m; b += blockDim.x) {
                const int64_t pp = b + tid;
                unsigned long long key = KEY_NONE;
                uint64_t v = 0;
                int64_t sp = pp;
                if (pp < m) {
                    sp = omap_get(s_om, pp);
                    v = ldw(A.w + ldi(pmap + sp) * stride + wl);
                    for (int l = 0; l < tt; ++l)
                        if ((v >> s_q[l]) & 1ull) v ^= s_u[l];
                    uint64_t z = v & (~0ull << c0);
                    if (lim < 64) z &= (1ull << lim) - 1;
                    if (z)
                        key = (static_cast<unsigned long long>(__ffsll(static_cast<long long>(z)) - 1) << 48) |
                              static_cast<unsigned long long>(pp - ob);
                }
                int myidx = -1;
                if (build && v != 0) {
                    myidx = atomicAdd(&s_cn, 1);
                    if (myidx < cap) {
                        c_w[myidx] = v;
                        c_pos[myidx] = static_cast<int>(pp - base);
                        c_src[myidx] = static_cast<int>(sp - base);
                        c_tt[myidx] = static_cast<uint8_t>(tt);
                    }
                }
                unsigned long long k = warp_min64(key);
                if (lane == 0) s_red[warp] = k;
                __syncthreads();
                if (warp == 0) {
                    unsigned long long kk = lane < nwarps ? s_red[lane] : KEY_NONE;
                    kk = warp_min64(kk);
                    if (lane == 0 && kk < s_best) s_best = kk;
                }
                __syncthreads();
                const unsigned long long bk = s_best;
                if (key != KEY_NONE && key == bk) {
                    s_bword = v;
                    s_bsrc = sp;
                    s_bidx = myidx;
                }
                if (bk != KEY_NONE) {
                    const int bc = static_cast<int>(bk >> 48);
                    if (bc == c0 && !build) break;
                    lim = bc;
                }
            }
            __syncthreads();
            if (build && tid == 0) s_cstate = s_cn <= cap && m - ob < (1 << 24) ? 1 : 2;
            __syncthreads();
        }

        if (warp == 0) {
            const unsigned long long bk = s_best;
            const int lim = s_lim;
            const int pr = p - bb;
            if (bk != KEY_NONE && static_cast<int>(bk >> 48) < lim) {
                // the outside row enters at p; the content of p leaves for pstar
                const int cstar = static_cast<int>(bk >> 48);
                const int64_t pstar = ob + static_cast<int64_t>(bk & ((1ull << 48) - 1));
                const uint64_t u = s_bword;
                const int psrc = __shfl_sync(FULL, src, pr);
                const uint64_t wpr = __shfl_sync(FULL, w, pr);
                if (lane == pr) {
                    w = u;
                    src = static_cast<int>(s_bsrc - base);
                }
                if (lane == 0 && s_cstate == 1) {  // pstar's list entry now holds p's row (t pivots applied)
                    const int bi = s_bidx;
                    c_w[bi] = wpr;
                    c_src[bi] = psrc;
                    c_tt[bi] = static_cast<uint8_t>(t);
                }
                if (lane == 0) {
                    omap_put(s_om, pstar, base + psrc);
                    s_om_pos[s_nom] = pstar;
                    s_nom = s_nom + 1;
                }
                record_pivot(cstar, u, pstar);
                const uint64_t us = u & above(cstar);
                if (lane > pr && ((w >> cstar) & 1ull)) w ^= us;
                ++t;
                ++p;
                col = cstar + 1;
            } else if (lim < 64) {
                // columns [col, lim) are zero everywhere: pivot in the window at column lim
                const int cstar = lim;
                const unsigned hit = __ballot_sync(FULL, lane >= pr && ((w >> cstar) & 1ull));
                const int ln = __ffs(hit) - 1;
                const uint64_t u = __shfl_sync(FULL, w, ln);
                const uint64_t wp = __shfl_sync(FULL, w, pr);
                const int usrc = __shfl_sync(FULL, src, ln);
                const int psrc = __shfl_sync(FULL, src, pr);
                if (lane == ln) {
                    w = wp;
                    src = psrc;
                }
                if (lane == pr) {
                    w = u;
                    src = usrc;
                }
                record_pivot(cstar, u, base + bb + ln);
                const uint64_t us = u & above(cstar);
                if (lane > pr && ((w >> cstar) & 1ull)) w ^= us;
                ++t;
                ++p;
                col = cstar + 1;
            } else {
                col = 64;  // nothing left in this leaf
            }
        }
        __syncthreads();
    }

    // ---- outputs: re-map the moved positions (pmap[dst] <- pmap[pre-leaf source]),
    // write the pivot rows' final leaf words, publish the pivots
    F2_STAMP(st, 11);
    F2_MARK(3);
    if (warp == 0) {
        record_moves(bb + lane < span && src != bb + lane, bb + lane, src);
        // the outside positions that received another row (first occurrence of each; the ones
        // the window absorbed were recorded above), across the warp in list order
        const int nom = s_nom;
        for (int i0 = 0; i0 < nom; i0 += 32) {
            const int i = i0 + lane;
            bool keep = false;
            int64_t pp = 0, v = 0;
            if (i < nom) {
                pp = s_om_pos[i];
                if (pp >= base + bb + 32) {
                    bool dup = false;
                    for (int j = 0; j < i; ++j) dup |= (s_om_pos[j] == pp);
                    if (!dup) {
                        v = omap_get(s_om, pp);
                        keep = v != pp;
                    }
                }
            }
            const unsigned bm = __ballot_sync(FULL, keep);
            if (keep) {
                const int idx = nmv + __popc(bm & ((1u << lane) - 1));
                s_mv_dst[idx] = pp;
                s_mv_phys[idx] = pmap[v];
            }
            nmv += __popc(bm);
        }
        if (lane == 0) s_nmv = nmv;
    }
    __syncthreads();
    const int nmv_all = s_nmv;
    const int mv0 = first_in_panel ? 0 : st->nmoved;
    for (int i = tid; i < nmv_all; i += blockDim.x) {
        pmap[s_mv_dst[i]] = s_mv_phys[i];
        st->moved[mv0 + i] = s_mv_dst[i];
    }
    __syncthreads();
    const int kb = s_t;
    // pivot rows carry their final leaf word (L bits, leading 1, S bits) from here on
    for (int l = tid; l < kb; l += blockDim.x) A.w[pmap[base + l] * stride + wl] = s_uf[l];
    if (tid == 0) {
        st->nmoved = mv0 + nmv_all;
        st->pmap_hi = m;  // outside swaps may have re-mapped any position
        st->leaf_r = base;
        st->leaf_kb = kb;
        st->r = base + kb;
        uint64_t mask = 0;
        for (int l = 0; l < kb; ++l) mask |= 1ull << s_q[l];
        st->leaf_mask = mask;
        const int64_t pkb = first_in_panel ? 0 : st->panel_kb;
        if (first_in_panel) st->panel_r = base;
        for (int l = 0; l < kb; ++l) {
            st->panel_q[pkb + l] = leaf_in_panel * 64 + s_q[l];
            st->brow[leaf_in_panel * 64 + s_q[l]] = base + l;
        }
        st->panel_kb = pkb + kb;
    }
    F2_STAMP(st, 12);
    F2_MARK(4);
    for (int l = tid; l < 64; l += blockDim.x) {
        st->ustrict[l] = l < kb ? s_u[l] : 0ull;
        st->ufull[l] = l < kb ? s_uf[l] : 0ull;
        st->q[l] = l < kb ? s_q[l] : 64;
    }
}

}  // namespace f2g
