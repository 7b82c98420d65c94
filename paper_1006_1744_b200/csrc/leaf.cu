// Leaf of the PLS engine: one 64-column word of the panel.
//
//   k_leaf_pivot    exact Gaussian pivot search on the leaf word (1 CTA)
//   k_row_moves     applies the leaf's row transpositions to whole rows
//   k_leaf_finalize eliminates the leaf word of every row >= leaf_r
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
__device__ __forceinline__ int64_t pick(const int64_t (&v)[S], int s) {
    int64_t r = v[0];
#pragma unroll
    for (int i = 1; i < S; ++i)
        if (s == i) r = v[i];
    return r;
}

}  // namespace

// One CTA of 1024 threads.  Warp 0 keeps a window of the first 128 positions
// of the leaf (r .. r+127) in registers, eagerly eliminated, and finds pivots
// there without any block-level synchronisation.  The window is exact whenever
// the leftmost nonzero column among its candidates equals the next unprocessed
// column (it then cannot be beaten, and window positions precede all others).
// Otherwise the whole block scans the positions past the window, catching each
// row up on the pivots found so far, for the leftmost column below the window's
// candidate (SURVEY.md §7 "Hard parts" 1).
__global__ void __launch_bounds__(1024, 1)
k_leaf_pivot(Mat A, int64_t wl, int lw, int first_in_panel, int leaf_in_panel, int panel_bits,
             PlsState* st, int64_t* P, int64_t* Qp) {
    constexpr int S = kWinSlots;
    __shared__ uint64_t s_u[64];
    __shared__ int s_q[64];
    __shared__ Omap s_om;
    __shared__ unsigned long long s_red[32];
    __shared__ unsigned long long s_best;
    __shared__ uint64_t s_bword;
    __shared__ int64_t s_bsrc;
    __shared__ int s_cmd, s_col, s_lim, s_t;
    __shared__ int s_nom;
    __shared__ int64_t s_om_pos[64];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int64_t m = A.m, stride = A.stride;
    const int64_t base = st->r;
    const int64_t ob = base + kWin;  // first position outside the window

    for (int i = tid; i < kOmapSlots; i += blockDim.x) s_om.key[i] = -1;
    if (first_in_panel)
        for (int i = tid; i < panel_bits; i += blockDim.x) st->brow[i] = -1;
    if (tid == 0) s_nom = 0;
    __syncthreads();

    // warp-0 register window
    uint64_t wv[S];
    int64_t src[S];
    int t = 0, col = 0;
    int64_t pos = base;
    if (warp == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            int64_t p = base + lane + 32 * s;
            wv[s] = p < m ? A.w[p * stride + wl] : 0ull;
            src[s] = p;
        }
    }

    // swap position `pos` with window slot (ls, ss) / bring in an outside word,
    // record the pivot and eliminate the window below it
    auto take_pivot = [&](int cstar, uint64_t u, int64_t usrc, int64_t pstar, bool from_window,
                          int ln, int sl) {
        const int ps = static_cast<int>((pos - base) >> 5), pl = static_cast<int>((pos - base) & 31);
        uint64_t vpos = __shfl_sync(FULL, pick<S>(wv, ps), pl);
        int64_t spos = __shfl_sync(FULL, pick<S>(src, ps), pl);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (from_window && lane == ln && s == sl) {
                wv[s] = vpos;
                src[s] = spos;
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (lane == pl && s == ps) {
                wv[s] = u;
                src[s] = usrc;
            }
        }
        const uint64_t us = u & above(cstar);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            int64_t p = base + lane + 32 * s;
            if (p > pos && p < m && ((wv[s] >> cstar) & 1ull)) wv[s] ^= us;
        }
        if (lane == 0) {
            s_u[t] = us;
            s_q[t] = cstar;
            P[pos] = pstar;
            Qp[pos] = wl * 64 + cstar;
            if (!from_window) {
                omap_put(s_om, pstar, spos);
                s_om_pos[s_nom] = pstar;
                s_nom = s_nom + 1;
            }
        }
        __syncwarp();
        ++t;
        ++pos;
        col = cstar + 1;
    };

    while (true) {
        if (warp == 0) {
            int cmd = 0, lim = 64;
            while (true) {
                if (pos >= m || col >= lw) {
                    cmd = 0;
                    break;
                }
                const uint64_t cmask = ~0ull << col;
                uint64_t orv = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    int64_t p = base + lane + 32 * s;
                    if (p >= pos && p < m) orv |= wv[s] & cmask;
                }
                const uint64_t any = warp_or64(orv);
                const int cstar = any ? __ffsll(static_cast<long long>(any)) - 1 : 64;
                if (ob < m && cstar != col) {  // rows past the window may hold an earlier column
                    cmd = 1;
                    lim = cstar;
                    break;
                }
                if (!any) {
                    cmd = 0;
                    break;
                }
                int sl = -1, ln = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    int64_t p = base + lane + 32 * s;
                    unsigned b = __ballot_sync(FULL, p >= pos && p < m && ((wv[s] >> cstar) & 1ull));
                    if (sl < 0 && b) {
                        sl = s;
                        ln = __ffs(b) - 1;
                    }
                }
                const uint64_t u = __shfl_sync(FULL, pick<S>(wv, sl), ln);
                const int64_t usrc = __shfl_sync(FULL, pick<S>(src, sl), ln);
                take_pivot(cstar, u, usrc, base + ln + 32 * sl, true, ln, sl);
            }
            if (lane == 0) {
                s_cmd = cmd;
                s_col = col;
                s_lim = lim;
                s_t = t;
            }
        }
        __syncthreads();
        if (s_cmd == 0) break;

        // ---- block-wide scan of positions [ob, m) for the leftmost column in [col, lim)
        {
            const int c0 = s_col, tt = s_t;
            int lim = s_lim;
            if (tid == 0) s_best = KEY_NONE;
            __syncthreads();
            for (int64_t b = ob; b < m; b += blockDim.x) {
                const int64_t p = b + tid;
                unsigned long long key = KEY_NONE;
                uint64_t w = 0;
                int64_t sp = p;
                if (p < m) {
                    sp = omap_get(s_om, p);
                    w = A.w[sp * stride + wl];
                    for (int l = 0; l < tt; ++l)
                        if ((w >> s_q[l]) & 1ull) w ^= s_u[l];
                    uint64_t v = w & (~0ull << c0);
                    if (lim < 64) v &= (1ull << lim) - 1;
                    if (v)
                        key = (static_cast<unsigned long long>(__ffsll(static_cast<long long>(v)) - 1) << 48) |
                              static_cast<unsigned long long>(p - ob);
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
                    s_bword = w;
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
            if (bk != KEY_NONE && static_cast<int>(bk >> 48) < lim) {
                const int cstar = static_cast<int>(bk >> 48);
                const int64_t pstar = ob + static_cast<int64_t>(bk & ((1ull << 48) - 1));
                take_pivot(cstar, s_bword, s_bsrc, pstar, false, 0, 0);
            } else if (lim < 64) {
                // columns [col, lim) are zero everywhere: pivot in the window at column lim
                const int cstar = lim;
                int sl = -1, ln = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    int64_t p = base + lane + 32 * s;
                    unsigned b = __ballot_sync(FULL, p >= pos && p < m && ((wv[s] >> cstar) & 1ull));
                    if (sl < 0 && b) {
                        sl = s;
                        ln = __ffs(b) - 1;
                    }
                }
                const uint64_t u = __shfl_sync(FULL, pick<S>(wv, sl), ln);
                const int64_t usrc = __shfl_sync(FULL, pick<S>(src, sl), ln);
                take_pivot(cstar, u, usrc, base + ln + 32 * sl, true, ln, sl);
            } else {
                col = 64;  // nothing left in this leaf
            }
        }
        __syncthreads();
    }

    // ---- outputs
    if (warp == 0) {
        const int kb = t;
        int n_out = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            int64_t p = base + lane + 32 * s;
            bool moved = p < m && src[s] != p;
            unsigned b = __ballot_sync(FULL, moved);
            if (moved) {
                int idx = n_out + __popc(b & ((1u << lane) - 1));
                st->swap_dst[idx] = p;
                st->swap_src[idx] = src[s];
            }
            n_out += __popc(b);
        }
        if (lane == 0) {
            for (int i = 0; i < s_nom; ++i) {
                int64_t p = s_om_pos[i];
                bool dup = false;
                for (int j = 0; j < i; ++j) dup |= (s_om_pos[j] == p);
                if (dup) continue;
                int64_t v = omap_get(s_om, p);
                if (v != p) {
                    st->swap_dst[n_out] = p;
                    st->swap_src[n_out] = v;
                    ++n_out;
                }
            }
            st->nswap = n_out;
            st->leaf_r = base;
            st->leaf_kb = kb;
            st->r = base + kb;
            uint64_t mask = 0;
            for (int l = 0; l < kb; ++l) mask |= 1ull << s_q[l];
            st->leaf_mask = mask;
            int64_t pkb = first_in_panel ? 0 : st->panel_kb;
            if (first_in_panel) st->panel_r = base;
            for (int l = 0; l < kb; ++l) {
                st->panel_q[pkb + l] = leaf_in_panel * 64 + s_q[l];
                st->brow[leaf_in_panel * 64 + s_q[l]] = base + l;
            }
            st->panel_kb = pkb + kb;
        }
        for (int l = lane; l < 64; l += 32) {
            st->ustrict[l] = l < kb ? s_u[l] : 0ull;
            st->q[l] = l < kb ? s_q[l] : 64;
        }
    }
}

// Row moves of one leaf: position swap_dst[i] receives the pre-leaf content of
// physical row swap_src[i].  The sets of destinations and sources coincide, so
// every CTA stages its column slice of all sources before writing.
__global__ void __launch_bounds__(256)
k_row_moves(Mat A, int64_t nwords, const PlsState* st) {
    extern __shared__ uint64_t s_buf[];  // [kMaxSwaps][32]
    const int ns = st->nswap;
    if (ns == 0) return;
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int nw = static_cast<int>(nwords - w0 < 32 ? nwords - w0 : 32);
    for (int i = threadIdx.x; i < ns * 32; i += blockDim.x) {
        int e = i >> 5, k = i & 31;
        if (k < nw) s_buf[i] = A.w[st->swap_src[e] * A.stride + w0 + k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ns * 32; i += blockDim.x) {
        int e = i >> 5, k = i & 31;
        if (k < nw) A.w[st->swap_dst[e] * A.stride + w0 + k] = s_buf[i];
    }
}

// Eliminate the leaf word of every row at position >= leaf_r: the row at
// position leaf_r + t (t < kb) is pivot row t and takes pivots l < t; every
// other row takes all kb pivots.  Afterwards a non-pivot row's leaf word holds
// exactly its L coefficients at the pivot columns (gauss.cpp:47-49).
__global__ void __launch_bounds__(256)
k_leaf_finalize(Mat A, int64_t wl, const PlsState* st) {
    __shared__ uint64_t su[64];
    __shared__ int sq[64];
    const int64_t kb = st->leaf_kb, r0 = st->leaf_r;
    if (kb == 0) return;
    if (threadIdx.x < 64) {
        su[threadIdx.x] = st->ustrict[threadIdx.x];
        sq[threadIdx.x] = st->q[threadIdx.x];
    }
    __syncthreads();
    for (int64_t p = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < A.m;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t* wp = A.w + p * A.stride + wl;
        uint64_t w = *wp;
        const int tl = static_cast<int>(p - r0 < kb ? p - r0 : kb);
        for (int l = 0; l < tl; ++l)
            if ((w >> sq[l]) & 1ull) w ^= su[l];
        *wp = w;
    }
}

void launch_leaf_pivot(cudaStream_t s, const Mat& A, int64_t wl, int lw, int first, int leaf_in_panel,
                       int panel_bits, PlsState* st, int64_t* P, int64_t* Qp) {
    k_leaf_pivot<<<1, 1024, 0, s>>>(A, wl, lw, first, leaf_in_panel, panel_bits, st, P, Qp);
}

void launch_row_moves(cudaStream_t s, const Mat& A, int64_t nwords, const PlsState* st) {
    const int grid = static_cast<int>((nwords + 31) / 32);
    const size_t smem = sizeof(uint64_t) * kMaxSwaps * 32;
    k_row_moves<<<grid, 256, smem, s>>>(A, nwords, st);
}

void launch_leaf_finalize(cudaStream_t s, const Mat& A, int64_t wl, const PlsState* st, int nsm) {
    int64_t blocks = (A.m + 255) / 256;
    int grid = static_cast<int>(blocks < 4 * nsm ? blocks : 4 * nsm);
    if (grid < 1) grid = 1;
    k_leaf_finalize<<<grid, 256, 0, s>>>(A, wl, st);
}

void setup_leaf_kernels() {
    cudaFuncSetAttribute(k_row_moves, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(uint64_t) * kMaxSwaps * 32));
}

}  // namespace f2g
