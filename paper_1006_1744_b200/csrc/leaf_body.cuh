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
__device__ __forceinline__ uint32_t pick(const uint32_t (&v)[S], int s) {
    uint32_t r = v[0];
#pragma unroll
    for (int i = 1; i < S; ++i)
        if (s == i) r = v[i];
    return r;
}

template <bool B>
struct BoolC {
    static constexpr bool value = B;
};

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
// The first 128 positions of the current order ("the window", a prefix of that order) decide
// a leaf whenever every column finds its pivot among them: row_pivots below applies the
// Gaussian pivot rule (gauss.cpp:33-49) to the window's leaf words in registers.  A column
// without candidates is decided only when no rows lie past the window; otherwise the leaf
// falls back to the general search further down (rank-deficient / sparse inputs).
//
// The panel kernel (panel.cu, pipe_fast_leaf) drives this on its carried 128-row window and
// then solves the pivot rows over the rest of the panel.
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
    uint4 stp[64];               // pivot steps as the search stores them: word lo, hi, source slot | column << 8 |
                                 // position << 16, -
    uint64_t linv[64];           // rows of L11^{-1} over pivot indices
    int posc[64];                // leaf column -> pivot index, -1
    int step_p[64], step_c[64];  // pivot steps: position in the order at the step, column
    int src[128];                // slot s now holds the pre-leaf content of slot src[s]
    uint64_t uf[64];             // pivot rows' final leaf words
    int wcount[4];
    int final_kb;                // -1: fell back
    int used4;                   // the 96-slot pass could not decide, all 128 slots searched
    uint64_t fbas[64];           // finalize basis
    uint64_t cfin[64];           // pivot rows' leaf words transposed (bit l = row l's bit in column c)
    uint32_t ainv[32], brows[32];
#ifdef F2_LEAF_CLOCKS
    long long clk[2];            // search loop start / end
#endif
};

// Warp 0: the same pivot rule in ROW form.  Lane l keeps the leaf words of window slots
// l, l+32, l+64, l+96 in registers (two 32-bit halves each) together with each row's
// current position in the order.  Per column: every row with a 1 there offers the key
// (position, row id); one hardware min-reduction picks the first row in the current order
// (gauss.cpp:33-40), two shuffles fetch its word, the other offering rows add it from the
// next column on (gauss.cpp:47-49), the row that sat at position t takes the pivot's old
// position (the transposition, :44) and the pivot row retires (its word is final: it
// holds the L bits left of each pivot column and U from the column on).  The dependent
// chain per pivot is one reduction and one shuffle round, one warp, no cross-warp protocol
// (the column-form search it replaces -- 128-bit slot masks per column, a lowest-bit carry
// chain, a second warp replaying every published step and a third tracking the slot
// permutation -- took 14.4K cycles per 64-column leaf; this one 10.7K).
// wsrc = the leaf word of slot 0, slots 16 words apart.
// Fills step_c/step_p, posc, uf, src (every slot) and final_kb (-1: a column without candidates
// in the window while rows lie past it).  NR = 3 searches the first 96 slots only (a quarter
// less work per column; the caller repeats the search on all 128 when that cannot decide).
template <int NR>
__device__ __forceinline__ int row_pivots(FastSmem& F, const uint64_t* wsrc, int lw, bool more) {
    const int lane = threadIdx.x & 31;
    uint32_t lo[NR], hi[NR], kp[NR];  // kp: position << 7 | row id (j << 5 | lane); ~0 once retired
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const uint64_t w = wsrc[(32 * j + lane) * 16];
        lo[j] = static_cast<uint32_t>(w);
        hi[j] = static_cast<uint32_t>(w >> 32);
        kp[j] = (static_cast<uint32_t>(32 * j + lane) << 7) | static_cast<uint32_t>(32 * j + lane);
    }
    int t = 0;
    const uint32_t stp_a = static_cast<uint32_t>(__cvta_generic_to_shared(&F.stp[0]));
    // One column: cb = its bit in the half holding it, am = the bits above it in that half.
    // Branch-free: a column without candidates is a masked no-op step (after a column the
    // window cannot decide the later steps still run, and the leaf is discarded).
    auto column = [&](auto hi_half, int c, uint32_t cb, uint32_t am) {
        constexpr bool HI = decltype(hi_half)::value;
        uint32_t key[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j) key[j] = ((HI ? hi[j] : lo[j]) & cb) ? kp[j] : ~0u;
        // this lane's first candidate and its word (selected beside the reduction)
        const bool s01 = key[1] < key[0];
        const uint32_t k01 = s01 ? key[1] : key[0];
        uint32_t k23 = key[2], l23 = lo[2], h23 = hi[2];
        if constexpr (NR == 4) {
            const bool s23 = key[3] < key[2];
            k23 = s23 ? key[3] : key[2];
            l23 = s23 ? lo[3] : lo[2];
            h23 = s23 ? hi[3] : hi[2];
        }
        const bool sb = k23 < k01;
        const uint32_t km = __reduce_min_sync(FULL, sb ? k23 : k01);
        const uint32_t blo = sb ? l23 : (s01 ? lo[1] : lo[0]);
        const uint32_t bhi = sb ? h23 : (s01 ? hi[1] : hi[0]);
        const uint32_t plo = __shfl_sync(FULL, blo, km & 31), phi = __shfl_sync(FULL, bhi, km & 31);
        const bool some = km != ~0u;
        const uint32_t p7 = km & ~127u;
        const uint32_t kmx = some ? km : 0xfffffffeu;  // no pivot: nothing equals it
        const uint32_t tk = some ? static_cast<uint32_t>(t) << 7 : 0xfffffffeu;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const bool cand = key[j] != ~0u, piv = key[j] == kmx;
            const uint32_t amj = piv ? ~0u : am;  // the pivot row adds itself: cleared, it never offers again
            if (!HI && cand) lo[j] ^= plo & amj;
            if (cand) hi[j] ^= HI ? phi & amj : phi;
            if ((kp[j] & ~127u) == tk) kp[j] = (kp[j] & 127u) | p7;  // slot t's row moves to p
            if (piv) kp[j] = ~0u;
        }
        // every lane stores the same 16 bytes (predicated on a pivot, shared-window address
        // computed once outside the loop)
        asm volatile(
            "{\n\t.reg .pred q;\n\t"
            "setp.ne.u32 q, %0, 0xffffffff;\n\t"
            "@q st.shared.v4.u32 [%1], {%2, %3, %4, %5};\n\t}" ::"r"(km),
            "r"(stp_a + 16u * t), "r"(plo), "r"(phi),
            "r"((km & 127u) | (static_cast<uint32_t>(c) << 8) | (p7 << 9)), "r"(0u)
            : "memory");
        t += some ? 1 : 0;
    };
    int ncol = 0;
    F2_CLK(if (lane == 0) F.clk[0] = clock64();)
    // blocks of 8 columns without a branch inside; between blocks, stop once a column could
    // not be decided (the pass is discarded anyway)
    {
        const int c1 = lw < 32 ? lw : 32;
        uint32_t cb = 1u, am = ~1u;
        int c = 0;
        for (; c + 8 <= c1 && !(more && t < c); c += 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i, cb <<= 1, am <<= 1) column(BoolC<false>{}, c + i, cb, am);
        }
        if (c + 8 > c1)
            for (; c < c1; ++c, cb <<= 1, am <<= 1) column(BoolC<false>{}, c, cb, am);
        ncol = c1;
    }
    {
        uint32_t cb = 1u, am = ~1u;
        int c = 32;
        for (; c + 8 <= lw && !(more && t < c); c += 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i, cb <<= 1, am <<= 1) column(BoolC<true>{}, c + i, cb, am);
        }
        if (c + 8 > lw)
            for (; c < lw; ++c, cb <<= 1, am <<= 1) column(BoolC<true>{}, c, cb, am);
        if (lw > 32) ncol = lw;
    }
    F2_CLK(if (lane == 0) F.clk[1] = clock64();)
    const bool ok = !(more && t < ncol);
    F.posc[lane] = -1;
    F.posc[lane + 32] = -1;
    __syncwarp();
    for (int l = lane; l < t; l += 32) {
        const uint4 e = F.stp[l];
        const uint32_t pk = e.z;
        F.uf[l] = e.x | (static_cast<uint64_t>(e.y) << 32);
        F.src[l] = static_cast<int>(pk & 127u);
        F.step_c[l] = static_cast<int>((pk >> 8) & 63u);
        F.step_p[l] = static_cast<int>(pk >> 16);
        F.posc[(pk >> 8) & 63u] = l;
    }
    if (ok) {
#pragma unroll
        for (int j = 0; j < NR; ++j)
            if (kp[j] != ~0u) F.src[kp[j] >> 7] = static_cast<int>(kp[j] & 127u);  // rows left: positions t..
        if (NR == 3) F.src[96 + lane] = 96 + lane;  // (not searched: they stay)
    }
    if (lane == 0) F.final_kb = ok ? t : -1;
    return ok ? t : -1;  // (uniform)
}

// Warps 0 and 1 after row_pivots: rows of L11^{-1} in pivot-index coordinates.  Row l's L
// bits in pivot order are bits q_0, q_1, ... of its final word: with 64 pivots in a 64-column
// leaf (q_t = t) the word itself; otherwise the words are transposed into column form
// (F.cfin: bit l of column c = row l's bit there) and the pivot columns transposed back.
// Then L11 = [A 0; B C] in 32x32 blocks: A^{-1} (warp 0) and C^{-1} (warp 1) by 32-step
// shuffle chains in parallel, and the off-diagonal block C^{-1} B A^{-1} by two independent
// passes.
__device__ __forceinline__ void pair_linv_rows(FastSmem& F, int kb) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t rows, rowsb = 0;
    if (kb == 64) {
        const uint64_t u1 = F.uf[lane + 32];
        if (w == 0) {
            rows = static_cast<uint32_t>(F.uf[lane]) & ((1u << lane) - 1u);  // A rows
            rowsb = static_cast<uint32_t>(u1);                               // B rows
        } else {
            rows = static_cast<uint32_t>(u1 >> 32) & ((1u << lane) - 1u);    // C rows
        }
    } else {
        const uint32_t r0 = warp_transpose32(static_cast<uint32_t>((lane < kb ? F.uf[lane] : 0ull) >> (32 * w)), lane);
        const uint32_t r1 =
            warp_transpose32(static_cast<uint32_t>((lane + 32 < kb ? F.uf[lane + 32] : 0ull) >> (32 * w)), lane);
        F.cfin[32 * w + lane] = r0 | (static_cast<uint64_t>(r1) << 32);
        asm volatile("bar.sync 2, 64;\n" ::: "memory");
        const int tt = 32 * w + lane;
        const uint64_t vt = tt < kb ? F.cfin[F.step_c[tt]] : 0ull;  // bit l: L[l][tt] (for l > tt)
        if (w == 0) {
            rows = warp_transpose32(static_cast<uint32_t>(vt), lane) & ((1u << lane) - 1u);
            rowsb = warp_transpose32(static_cast<uint32_t>(vt >> 32), lane);
        } else {
            (void)warp_transpose32(static_cast<uint32_t>(vt), lane);
            rows = warp_transpose32(static_cast<uint32_t>(vt >> 32), lane) & ((1u << lane) - 1u);
        }
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
