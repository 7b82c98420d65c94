// Leaf of the PLS engine: one 64-column word of the panel.
//
//   k_leaf_pivot    exact Gaussian pivot search on the leaf word (1 CTA); the
//                   leaf's transpositions only re-map positions (pmap)
//   k_perm_save/put at the end of a panel, the panel's transpositions applied to
//                   whole rows in one gather
//
// Bit-exactness rests on the pivot rule of gauss_pls (proj/src/gauss.cpp:33-49):
// the pivot is the leftmost column that has a nonzero at or below position r,
// and in it the first row in the *current* row order; P[r] = that position,
// Q[r] = that column; rows r and P[r] are swapped as a transposition; rows below
// are cleared starting one column right of the pivot so the L bit stays.  Only
// the leaf word's bits decide pivots in the leaf's columns, so the search reads
// one word per row (the restructuring SURVEY.md §7 "Hard parts" 2 validates).
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned long long KEY_NONE = ~0ull;

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
    uint32_t lo = __reduce_or_sync(FULL, static_cast<uint32_t>(v));
    uint32_t hi = __reduce_or_sync(FULL, static_cast<uint32_t>(v >> 32));
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ unsigned long long warp_min64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
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
__global__ void __launch_bounds__(1024, 1)
k_leaf_pivot(Mat A, int64_t wl, int lw, int first_in_panel, int leaf_in_panel, int panel_bits,
             PlsState* st, int64_t* P, int64_t* Qp, int64_t* pmap, int64_t qcol_off) {
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
        wo = catch_up(A.w[pmap[sabs] * stride + wl], tt);
    };
    // raw pre-leaf word of relative position x, loaded early for the next slide
    uint64_t pf_w = 0;
    auto prefetch = [&](int x) { pf_w = x < span ? A.w[pmap[base + x] * stride + wl] : 0ull; };

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

        // ---- block-wide scan of positions [ob, m) for the leftmost column in [col, lim)
        const int64_t ob = base + s_ob;
        {
            const int c0 = s_col, tt = s_t;
            int lim = s_lim;
            if (tid == 0) s_best = KEY_NONE;
            __syncthreads();
            for (int64_t b = ob; b < m; b += blockDim.x) {
                const int64_t pp = b + tid;
                unsigned long long key = KEY_NONE;
                uint64_t v = 0;
                int64_t sp = pp;
                if (pp < m) {
                    sp = omap_get(s_om, pp);
                    v = A.w[pmap[sp] * stride + wl];
                    for (int l = 0; l < tt; ++l)
                        if ((v >> s_q[l]) & 1ull) v ^= s_u[l];
                    uint64_t z = v & (~0ull << c0);
                    if (lim < 64) z &= (1ull << lim) - 1;
                    if (z)
                        key = (static_cast<unsigned long long>(__ffsll(static_cast<long long>(z)) - 1) << 48) |
                              static_cast<unsigned long long>(pp - ob);
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
                }
                if (bk != KEY_NONE) {
                    const int bc = static_cast<int>(bk >> 48);
                    if (bc == c0) break;
                    lim = bc;
                }
            }
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
                if (lane == pr) {
                    w = u;
                    src = static_cast<int>(s_bsrc - base);
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
    F2_MARK(3);
    if (warp == 0) {
        record_moves(bb + lane < span && src != bb + lane, bb + lane, src);
        if (lane == 0) {
            for (int i = 0; i < s_nom; ++i) {
                const int64_t pp = s_om_pos[i];
                if (pp < base + bb + 32) continue;  // absorbed by the window: recorded above
                bool dup = false;
                for (int j = 0; j < i; ++j) dup |= (s_om_pos[j] == pp);
                if (dup) continue;
                const int64_t v = omap_get(s_om, pp);
                if (v != pp) {
                    s_mv_dst[nmv] = pp;
                    s_mv_phys[nmv] = pmap[v];
                    ++nmv;
                }
            }
            s_nmv = nmv;
        }
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
    F2_MARK(4);
    for (int l = tid; l < 64; l += blockDim.x) {
        st->ustrict[l] = l < kb ? s_u[l] : 0ull;
        st->ufull[l] = l < kb ? s_uf[l] : 0ull;
        st->q[l] = l < kb ? s_q[l] : 64;
    }
}

// Per 8-column group of the leaf word: the finalize table F[g][v] (correction the
// group's pivots apply to a word whose byte g reads v, sequentially as gauss_pls
// does) and the index map M[g][e] = xor_{b in e} R[b], R the rows of the group's
// inverse 8x8 L block (see trsm.cu).  k_leaf_update consumes both.  One thread per
// table entry (16 CTAs x 256).
__global__ void __launch_bounds__(256) k_leaf_tables(PlsState* st, int leaf_in_panel) {
    __shared__ uint64_t s_u[64], s_uf[64];
    __shared__ int s_q[64];
    __shared__ int s_gs[9];
    const int tid = threadIdx.x;
    const int kb = static_cast<int>(st->leaf_kb);
    if (kb == 0) return;
    if (tid < 64) {
        s_u[tid] = st->ustrict[tid];
        s_uf[tid] = st->ufull[tid];
        s_q[tid] = st->q[tid];
    }
    __syncthreads();
    if (tid <= 8) {
        int lo = 0;
        while (lo < kb && s_q[lo] < 8 * tid) ++lo;
        s_gs[tid] = lo;
    }
    __syncthreads();

    const int i = blockIdx.x * 256 + tid;
    const int which = i >> 11, g = (i >> 8) & 7, v = i & 255;
    const int g0 = s_gs[g], g1 = s_gs[g + 1];
    if (which == 0) {
        uint64_t x = static_cast<uint64_t>(v) << (8 * g), corr = 0;
        for (int l = g0; l < g1; ++l)
            if ((x >> s_q[l]) & 1ull) {
                x ^= s_u[l];
                corr ^= s_u[l];
            }
        st->leaf_F[g][v] = corr;
    } else {
        uint32_t Rb[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) Rb[b] = 0;
        for (int l = g0; l < g1; ++l) {
            const int sb = s_q[l] - 8 * g;
            const uint32_t c = static_cast<uint32_t>(s_uf[l] >> (8 * g)) & ((1u << sb) - 1u);
            uint32_t R = 1u << sb;
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if ((c >> b) & 1u) R ^= Rb[b];
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if (b == sb) Rb[b] = R;
        }
        uint32_t Mv = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if ((v >> b) & 1) Mv ^= Rb[b];
        st->leaf_M[g][v] = static_cast<uint8_t>(Mv);
    }
}

// Per leaf j of the finished panel (one CTA each, in parallel): the bytewise map
// c -> c * L_jj^{-1} of the leaf's 64x64 unit lower block, for k_panel_trsm.
// lmap[j][g][v] = xor over bits b of v of R(pivot at raw 64j+8g+b), R_l = e_{q_l} ^
// sum_{l'<l} c_l[l'] R_l' (c_l = pivot row l's L bits); built group by group, earlier
// groups through their finished byte maps.  Runs after the panel's row gather, so the
// pivot rows sit at physical positions panel_r + t.
__global__ void __launch_bounds__(256) k_panel_lmaps(Mat Cf, int64_t pw0, PlsState* st) {
    __shared__ uint64_t s_uf[64];
    __shared__ int s_q[64];
    __shared__ int s_gs[9];
    __shared__ int s_pos[64];
    __shared__ uint64_t s_R[64];
    __shared__ uint64_t s_L[8][256];
    const int j = blockIdx.x, tid = threadIdx.x;
    const int nk = static_cast<int>(st->panel_kb);
    const int64_t r0 = st->panel_r;
    __shared__ int s_t0, s_t1;
    if (tid == 0) {
        int lo = 0;
        while (lo < nk && st->panel_q[lo] < 64 * j) ++lo;
        int hi = lo;
        while (hi < nk && st->panel_q[hi] < 64 * j + 64) ++hi;
        s_t0 = lo;
        s_t1 = hi;
    }
    if (tid < 64) s_pos[tid] = -1;
    __syncthreads();
    const int t0 = s_t0, kb = s_t1 - s_t0;
    if (kb == 0) return;
    if (tid < kb) {
        s_q[tid] = st->panel_q[t0 + tid] - 64 * j;
        s_uf[tid] = Cf.w[(r0 + t0 + tid) * Cf.stride + pw0 + j];
    }
    __syncthreads();
    if (tid < kb) s_pos[s_q[tid]] = tid;
    if (tid <= 8) {
        int lo = 0;
        while (lo < kb && s_q[lo] < 8 * tid) ++lo;
        s_gs[tid] = lo;
    }
    __syncthreads();
    for (int g = 0; g < 8; ++g) {
        if (tid == 0) {
            for (int l = s_gs[g]; l < s_gs[g + 1]; ++l) {
                const uint64_t c = s_uf[l] & ((1ull << s_q[l]) - 1ull);
                uint64_t R = 1ull << s_q[l];
                for (int g2 = 0; g2 < g; ++g2) R ^= s_L[g2][(c >> (8 * g2)) & 0xffu];
                const unsigned inb = static_cast<unsigned>(c >> (8 * g)) & 0xffu;
                for (int b = 0; b < 8; ++b)
                    if ((inb >> b) & 1u) R ^= s_R[s_pos[8 * g + b]];
                s_R[l] = R;
            }
        }
        __syncthreads();
        uint64_t x = 0;
        for (int b = 0; b < 8; ++b) {
            const int l = s_pos[8 * g + b];
            if (((tid >> b) & 1) && l >= 0) x ^= s_R[l];
        }
        s_L[g][tid] = x;
        __syncthreads();
    }
    for (int g = 0; g < 8; ++g) st->lmap[j][g][tid] = s_L[g][tid];
}

void launch_panel_lmaps(cudaStream_t s, const Mat& Cf, int64_t pw0, int nleaves, PlsState* st) {
    k_panel_lmaps<<<nleaves, 256, 0, s>>>(Cf, pw0, st);
}

// ---- column-sharded (multi-GPU) panel exchange --------------------------------------
// Header of one factored panel (int64): [0] kb, [1] panel_r, [2] nmoved, [3] reserved,
// [4, 4+W) pivot columns (panel-relative), then kMaxMoved re-mapped positions, then
// their source rows (pmap values), then W entries P[panel_r + t].
__global__ void __launch_bounds__(256) k_dist_export(const PlsState* st, const int64_t* pmap, const int64_t* P,
                                                    int64_t* hdr, int W) {
    const int kb = static_cast<int>(st->panel_kb), nm = st->nmoved;
    const int64_t r0 = st->panel_r;
    int64_t* q = hdr + 4;
    int64_t* mv = q + W;
    int64_t* src = mv + kMaxMoved;
    int64_t* pp = src + kMaxMoved;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    if (tid == 0) {
        hdr[0] = kb;
        hdr[1] = r0;
        hdr[2] = nm;
        hdr[3] = 0;
    }
    for (int t = tid; t < kb; t += nth) {
        q[t] = st->panel_q[t];
        pp[t] = P[r0 + t];
    }
    for (int i = tid; i < nm; i += nth) {
        mv[i] = st->moved[i];
        src[i] = pmap[st->moved[i]];
    }
}

// A rank that does not own the panel adopts the owner's header: pivot bookkeeping
// for the TRSM/Schur kernels and the re-mapped positions for the row gather.
__global__ void __launch_bounds__(1024) k_dist_import(PlsState* st, int64_t* pmap, const int64_t* hdr, int W) {
    const int kb = static_cast<int>(hdr[0]), nm = static_cast<int>(hdr[2]);
    const int64_t r0 = hdr[1];
    const int64_t* q = hdr + 4;
    const int64_t* mv = q + W;
    const int64_t* src = mv + kMaxMoved;
    const int tid = threadIdx.x, nth = blockDim.x;
    for (int i = tid; i < W; i += nth) st->brow[i] = -1;
    __syncthreads();
    for (int t = tid; t < kb; t += nth) {
        st->panel_q[t] = static_cast<int32_t>(q[t]);
        st->brow[q[t]] = r0 + t;
    }
    for (int i = tid; i < nm; i += nth) {
        st->moved[i] = mv[i];
        pmap[mv[i]] = src[i];
    }
    if (tid == 0) {
        st->panel_kb = kb;
        st->panel_r = r0;
        st->r = r0 + kb;
        st->nmoved = nm;
    }
}

__global__ void k_set_r(PlsState* st, int64_t r) {
    st->r = r;
    st->panel_kb = 0;
    st->nmoved = 0;
}

void launch_dist_export(cudaStream_t s, const PlsState* st, const int64_t* pmap, const int64_t* P, int64_t* hdr, int W) {
    k_dist_export<<<32, 256, 0, s>>>(st, pmap, P, hdr, W);
}
void launch_dist_import(cudaStream_t s, PlsState* st, int64_t* pmap, const int64_t* hdr, int W) {
    k_dist_import<<<1, 1024, 0, s>>>(st, pmap, hdr, W);
}
void launch_set_r(cudaStream_t s, PlsState* st, int64_t r) { k_set_r<<<1, 1, 0, s>>>(st, r); }

// Panel end, step 1: copy the rows that the panel's positions now refer to
// (physical row pmap[x] for every re-mapped position x) into scratch, whole width.
__global__ void __launch_bounds__(256) k_perm_save(Mat A, int64_t nwords, const PlsState* st, const int64_t* pmap,
                                                  uint64_t* scratch) {
    const int n = st->nmoved;
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nwords) return;
    for (int i = blockIdx.y; i < n; i += gridDim.y)
        scratch[static_cast<int64_t>(i) * A.stride + k] = A.w[pmap[st->moved[i]] * A.stride + k];
}

// Panel end, step 2: physical row x <- saved content, pmap back to identity.
// This applies the panel's transpositions (perm.cpp:8-16) to every column.
__global__ void __launch_bounds__(256) k_perm_put(Mat A, int64_t nwords, const PlsState* st, int64_t* pmap,
                                                 const uint64_t* scratch) {
    const int n = st->nmoved;
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (int i = blockIdx.y; i < n; i += gridDim.y) {
        const int64_t x = st->moved[i];
        if (k < nwords) A.w[x * A.stride + k] = scratch[static_cast<int64_t>(i) * A.stride + k];
        if (k == 0) pmap[x] = x;
    }
}

__global__ void k_pmap_init(int64_t* pmap, int64_t m) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        pmap[i] = i;
}

void launch_leaf_pivot(cudaStream_t s, const Mat& A, int64_t wl, int lw, int first, int leaf_in_panel,
                       int panel_bits, PlsState* st, int64_t* P, int64_t* Qp, int64_t* pmap, int64_t qcol_off) {
    k_leaf_pivot<<<1, 1024, 0, s>>>(A, wl, lw, first, leaf_in_panel, panel_bits, st, P, Qp, pmap, qcol_off);
}

void launch_perm(cudaStream_t s, const Mat& A, int64_t nwords, const PlsState* st, int64_t* pmap, uint64_t* scratch) {
    dim3 grid(static_cast<unsigned>((nwords + 255) / 256), 64);
    k_perm_save<<<grid, 256, 0, s>>>(A, nwords, st, pmap, scratch);
    k_perm_put<<<grid, 256, 0, s>>>(A, nwords, st, pmap, scratch);
}

void launch_leaf_tables(cudaStream_t s, PlsState* st, int leaf_in_panel) {
    k_leaf_tables<<<16, 256, 0, s>>>(st, leaf_in_panel);
}

void launch_pmap_init(cudaStream_t s, int64_t* pmap, int64_t m) {
    int64_t g = (m + 255) / 256;
    if (g > 1024) g = 1024;
    if (g < 1) g = 1;
    k_pmap_init<<<static_cast<int>(g), 256, 0, s>>>(pmap, m);
}

void setup_leaf_kernels() {}

}  // namespace f2g
