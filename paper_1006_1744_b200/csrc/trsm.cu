// Pivot-row triangular solve over GF(2).
//
// X_t = B_t xor sum_{l<t} L[t][l] X_l for the kb pivot rows of a leaf/panel
// (or an explicit unit-lower L), i.e. B <- L^{-1} B as trsm_lower_left_unit
// does (proj/src/mul.cpp:109-131; the diagonal is implicit and everything on
// or above it ignored).  L is read in "raw" form: row t's coefficient for
// pivot l sits at the pivot's raw column q_l of its coefficient words, which
// is how the packed layout stores L before compress_columns (gauss.cpp:47-53).
//
// Blocking: each CTA owns kTW target words of all kb rows in SMEM and walks the
// raw columns 8 at a time (group g).  The group's <= 8 pivots sit at raw bit
// positions sb_l = q_l - 8g of the coefficient byte.  With R = rows of the
// group's inverse 8x8 L block (R_l = e_l ^ xor_{l'<l, c_l bit} R_l'), a table T
// over the group rows' *current* values and M(e) = xor_{b in e} R[b], every row
// t >= t0 of the group and after it becomes X_t ^= T[M(c_t)], c_t its coefficient
// byte (masked below its own pivot for the group's rows).  The M maps depend only
// on the pivot rows' coefficients, which this kernel never modifies, so all of
// them are prepared up front in parallel; each group then costs one table build
// and one lookup pass (two barriers) and no serial in-group solve.
#include <cstdint>
#include <cstdlib>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kTW = 8;                 // target words per CTA
constexpr int kMaxTrsmBits = 1024;     // pivots per solve (the host never passes more)
constexpr int kThreads = 512;
constexpr int kCwPer = kMaxTrsmBits / kThreads;  // coefficient rows staged per thread

}  // namespace

__global__ void __launch_bounds__(kThreads)
k_pivot_trsm(Mat A, int64_t coef_w0, int coef_words, int64_t tw0, int64_t tw1, const PlsState* st,
             PivotSet ps, Mat L) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int rows_cap = coef_words * 64, ngroups = coef_words * 8;
    uint64_t* X = smem;                                                   // [rows_cap][kTW]
    uint64_t* T = X + rows_cap * kTW;                                     // [256][kTW]
    uint64_t* cw = T + 256 * kTW;                                         // [rows_cap] current coefficient word
    int32_t* sq = reinterpret_cast<int32_t*>(cw + rows_cap);              // [rows_cap]
    int32_t* gstart = sq + rows_cap;                                      // [ngroups + 1]
    int16_t* posrow = reinterpret_cast<int16_t*>(gstart + ngroups + 8);   // [ngroups][8]
    uint8_t* Mall = reinterpret_cast<uint8_t*>(posrow + ngroups * 8);     // [ngroups][256]

    int64_t kb, r0;
    const int32_t* qsrc = nullptr;
    if (ps.mode == 0) {
        kb = st->leaf_kb;
        r0 = st->leaf_r;
        qsrc = st->q;
    } else if (ps.mode == 1) {
        kb = st->panel_kb;
        r0 = st->panel_r;
        qsrc = st->panel_q;
    } else {
        kb = ps.kb;
        r0 = ps.r0;
    }
    if (kb <= 1) return;
    const int64_t tb = tw0 + static_cast<int64_t>(blockIdx.x) * kTW;
    if (tb >= tw1) return;
    const int ntw = static_cast<int>(tw1 - tb < kTW ? tw1 - tb : kTW);
    const int tid = threadIdx.x, nth = blockDim.x;
    const int nk = static_cast<int>(kb);

    auto coef_word = [&](int t, int wi) -> uint64_t {
        return ps.mode == 2 ? L.w[static_cast<int64_t>(t) * L.stride + wi] : A.w[(r0 + t) * A.stride + coef_w0 + wi];
    };

    for (int t = tid; t < nk; t += nth) sq[t] = qsrc ? qsrc[t] : t;
    for (int i0 = tid; i0 < nk * kTW; i0 += 4 * nth) {
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * nth, t = i / kTW, j = i % kTW;
            v[u] = (i < nk * kTW && j < ntw) ? A.w[(r0 + t) * A.stride + tb + j] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u * nth < nk * kTW) X[i0 + u * nth] = v[u];
    }
    for (int i = tid; i < ngroups * 8; i += nth) posrow[i] = -1;
    __syncthreads();
    for (int g = tid; g <= ngroups; g += nth) {
        int lo = 0, hi = nk;  // first t with sq[t] >= 8g
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sq[mid] < 8 * g) lo = mid + 1;
            else hi = mid;
        }
        gstart[g] = lo;
    }
    for (int t = tid; t < nk; t += nth) posrow[(sq[t] >> 3) * 8 + (sq[t] & 7)] = static_cast<int16_t>(t);
    __syncthreads();
    // index maps M of every group
    for (int i = tid; i < ngroups * 256; i += nth) {
        const int g = i >> 8, e = i & 255;
        const int t0 = gstart[g], t1 = gstart[g + 1];
        uint32_t Mv = 0;
        if (t1 > t0) {
            uint32_t Rb[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) Rb[b] = 0;
            const int sh = 8 * (g & 7), base = 8 * g;
            for (int l = t0; l < t1; ++l) {
                const int sb = sq[l] - base;
                const uint32_t c = static_cast<uint32_t>(coef_word(l, g >> 3) >> sh) & ((1u << sb) - 1u);
                uint32_t R = 1u << sb;
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    if ((c >> b) & 1u) R ^= Rb[b];
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    if (b == sb) Rb[b] = R;
            }
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if ((e >> b) & 1) Mv ^= Rb[b];
        }
        Mall[i] = static_cast<uint8_t>(Mv);
    }
    uint64_t cwn[kCwPer];
#pragma unroll
    for (int u = 0; u < kCwPer; ++u) {
        const int t = tid + u * nth;
        cwn[u] = t < nk ? coef_word(t, 0) : 0ull;
    }

    const int lane = tid & 31, wq = lane & 3, rq = lane >> 2, wrp = tid >> 5;
    for (int g = 0; g < ngroups; ++g) {
        if ((g & 7) == 0) {
            // coefficient word g/8 of every pivot row (prefetched one word ahead)
            __syncthreads();
#pragma unroll
            for (int u = 0; u < kCwPer; ++u) {
                const int t = tid + u * nth;
                if (t < nk) cw[t] = cwn[u];
            }
            const int wn = (g >> 3) + 1;
            if (wn < coef_words) {
#pragma unroll
                for (int u = 0; u < kCwPer; ++u) {
                    const int t = tid + u * nth;
                    if (t < nk) cwn[u] = coef_word(t, wn);
                }
            }
        }
        __syncthreads();
        const int t0 = gstart[g], t1 = gstart[g + 1];
        if (t0 == t1) continue;
        const int sh = 8 * (g & 7), base = 8 * g;
        const uint8_t* Mg = Mall + g * 256;
        // table over the group rows' current values: thread = (word j, 4 entries)
        {
            const int j = tid % kTW;
            const int16_t* pr = posrow + g * 8;
            uint64_t v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int l = pr[b];
                v[b] = l >= 0 ? X[l * kTW + j] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = tid / kTW + 64 * u;
                uint64_t x = 0;
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    if ((e >> b) & 1) x ^= v[b];
                T[e * kTW + j] = x;
            }
        }
        __syncthreads();
        // rows >= t0: 4 lanes per row (16 B each), 8 rows per warp instruction, so the
        // X accesses are contiguous 512-B runs (conflict-free)
#pragma unroll 4
        for (int t = t0 + wrp * 8 + rq; t < nk; t += (nth / 32) * 8) {
            uint32_t cb = static_cast<uint32_t>(cw[t] >> sh) & 0xffu;
            if (t < t1) cb &= (1u << (sq[t] - base)) - 1u;
            const uint32_t idx = Mg[cb];
            uint4* xr = reinterpret_cast<uint4*>(X + t * kTW) + wq;
            const uint4 b = *(reinterpret_cast<const uint4*>(T + idx * kTW) + wq);
            uint4 a = *xr;
            a.x ^= b.x;
            a.y ^= b.y;
            a.z ^= b.z;
            a.w ^= b.w;
            *xr = a;
        }
    }
    __syncthreads();
    for (int i = tid; i < nk * kTW; i += nth) {
        const int t = i / kTW, j = i % kTW;
        if (j < ntw) A.w[(r0 + t) * A.stride + tb + j] = X[i];
    }
}

static size_t trsm_smem(int coef_words) {
    const size_t rows = static_cast<size_t>(coef_words) * 64, groups = static_cast<size_t>(coef_words) * 8;
    return sizeof(uint64_t) * (rows * kTW + 256 * kTW + rows) + sizeof(int32_t) * (rows + groups + 8) +
           sizeof(int16_t) * groups * 8 + 256 * groups;
}

void launch_pivot_trsm(cudaStream_t s, const Mat& A, int64_t coef_w0, int coef_words, int64_t tw0,
                       int64_t tw1, const PlsState* st, PivotSet ps, const Mat* L) {
    if (tw1 <= tw0) return;
    const int grid = static_cast<int>((tw1 - tw0 + kTW - 1) / kTW);
    Mat l = L ? *L : Mat{nullptr, 0, 0, 0};
    k_pivot_trsm<<<grid, kThreads, trsm_smem(coef_words), s>>>(A, coef_w0, coef_words, tw0, tw1, st, ps, l);
}


// Panel TRSM by leaf blocks.  The panel's pivot rows form 64-pivot blocks (one per
// leaf); the panel kernel (or k_panel_lmaps) left, per leaf j, the bytewise map c -> c * L_jj^{-1}
// (st->lmap[j]).  Block step j: 8 tables over block j's rows as they are now (raw
// positions 64j..64j+63), then every row t of block j and after it adds
// xor_g T_g[byte_g(M)] with M = c_t * L_jj^{-1} (c_t = its coefficients for block j,
// masked below its own pivot inside block j).  That equals forward substitution with
// the whole block (the block's rows come out solved, later rows get the block's
// solved rows), so the panel needs one step per leaf instead of one per 8 pivots.
// 512-bit column strips (kPTW8 = 8 words): one wave of CTAs at 64K columns, and every
// table entry / row slice is 64 B read by 4 lanes with 16-byte accesses (a 4-word
// version's 32-B entries read by single lanes conflicted).
namespace {
constexpr int kPTW8 = 8;
}

__global__ void __launch_bounds__(512, 1)
k_panel_trsm8(Mat A, Mat Cf, int64_t coef_w0, int nleaves, int64_t tw0, int64_t tw1, const PlsState* st) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int rows_cap = nleaves * 64;
    uint64_t* X = smem;                                               // [rows_cap][8]
    uint64_t* T = X + rows_cap * kPTW8;                               // [8][256][8]
    uint64_t* Lm = T + 8 * 256 * kPTW8;                               // [8][256]
    uint64_t* cw = Lm + 8 * 256;                                      // [rows_cap]
    int32_t* sq = reinterpret_cast<int32_t*>(cw + rows_cap);          // [rows_cap]
    int16_t* posrow = reinterpret_cast<int16_t*>(sq + rows_cap);      // [rows_cap]
    int32_t* bstart = reinterpret_cast<int32_t*>(posrow + rows_cap);  // [nleaves + 1]

    const int nk = static_cast<int>(st->panel_kb);
    const int64_t r0 = st->panel_r;
    if (nk <= 1) return;
    const int64_t tb = tw0 + static_cast<int64_t>(blockIdx.x) * kPTW8;
    if (tb >= tw1) return;
    const int ntw = static_cast<int>(tw1 - tb < kPTW8 ? tw1 - tb : kPTW8);
    const int tid = threadIdx.x;

    for (int t = tid; t < nk; t += 512) sq[t] = st->panel_q[t];
    for (int i = tid; i < rows_cap; i += 512) posrow[i] = -1;
    for (int i = tid; i < nk * kPTW8; i += 512) {
        const int t = i >> 3, j = i & 7;
        X[i] = j < ntw ? A.w[(r0 + t) * A.stride + tb + j] : 0ull;
    }
    __syncthreads();
    for (int t = tid; t < nk; t += 512) posrow[sq[t]] = static_cast<int16_t>(t);
    for (int j = tid; j <= nleaves; j += 512) {
        int lo = 0, hi = nk;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sq[mid] < 64 * j) lo = mid + 1;
            else hi = mid;
        }
        bstart[j] = lo;
    }
    __syncthreads();

    constexpr int kLmPer = 8 * 256 / 512, kCwPer = kMaxTrsmBits / 512;
    uint64_t pf_lm[kLmPer], pf_cw[kCwPer];
    auto prefetch = [&](int j) {
        if (j >= nleaves) return;
        const int t0 = bstart[j];
#pragma unroll
        for (int u = 0; u < kLmPer; ++u) pf_lm[u] = (&st->lmap[j][0][0])[tid + u * 512];
#pragma unroll
        for (int u = 0; u < kCwPer; ++u) {
            const int t = t0 + tid + u * 512;
            pf_cw[u] = t < nk ? Cf.w[(r0 + t) * Cf.stride + coef_w0 + j] : 0ull;
        }
    };
    prefetch(0);
    const int sub = tid & 3, grp = tid >> 2;  // update: 4 lanes per row, 16 B each
    for (int j = 0; j < nleaves; ++j) {
        const int t0 = bstart[j], t1 = bstart[j + 1];
        if (t0 == t1) {
            prefetch(j + 1);
            continue;
        }
#pragma unroll
        for (int u = 0; u < kLmPer; ++u) Lm[tid + u * 512] = pf_lm[u];
#pragma unroll
        for (int u = 0; u < kCwPer; ++u) {
            const int t = t0 + tid + u * 512;
            if (t < nk) cw[t] = pf_cw[u];
        }
        prefetch(j + 1);
        // 8 tables over block j's rows as they are now: thread = (table g, 16-B chunk wc,
        // low nibble el); a warp covers 8 consecutive entries x 64 B (conflict-free)
        {
            const int g = tid >> 6, wc = tid & 3, el = (tid >> 2) & 15;
            uint4 v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int l = posrow[64 * j + 8 * g + b];
                v[b] = l >= 0 ? *reinterpret_cast<const uint4*>(X + l * kPTW8 + 2 * wc) : make_uint4(0, 0, 0, 0);
            }
            uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((el >> b) & 1) {
                    x.x ^= v[b].x;
                    x.y ^= v[b].y;
                    x.z ^= v[b].z;
                    x.w ^= v[b].w;
                }
            uint64_t* tg = T + g * 256 * kPTW8 + 2 * wc;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k) {
                    const uint4 h = v[4 + ((k & 1) ? 0 : ((k & 2) ? 1 : ((k & 4) ? 2 : 3)))];
                    x.x ^= h.x;
                    x.y ^= h.y;
                    x.z ^= h.z;
                    x.w ^= h.w;
                }
                const int eh = k ^ (k >> 1);
                *reinterpret_cast<uint4*>(tg + (eh * 16 + el) * kPTW8) = x;
            }
        }
        __syncthreads();
        for (int t = t0 + grp; t < nk; t += 128) {
            uint64_t c = cw[t];
            if (t < t1) c &= (1ull << (sq[t] - 64 * j)) - 1ull;
            uint64_t M = 0;
#pragma unroll
            for (int g = 0; g < 8; ++g) M ^= Lm[g * 256 + ((c >> (8 * g)) & 0xffu)];
            uint4 a = *reinterpret_cast<const uint4*>(X + t * kPTW8 + 2 * sub);
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const uint4 b = *reinterpret_cast<const uint4*>(T + (g * 256 + ((M >> (8 * g)) & 0xffu)) * kPTW8 + 2 * sub);
                a.x ^= b.x;
                a.y ^= b.y;
                a.z ^= b.z;
                a.w ^= b.w;
            }
            *reinterpret_cast<uint4*>(X + t * kPTW8 + 2 * sub) = a;
        }
        __syncthreads();
    }
    for (int i = tid; i < nk * kPTW8; i += 512) {
        const int t = i >> 3, jj = i & 7;
        if (jj < ntw) A.w[(r0 + t) * A.stride + tb + jj] = X[i];
    }
}

static size_t panel_trsm8_smem(int nleaves) {
    const size_t rows = static_cast<size_t>(nleaves) * 64;
    return sizeof(uint64_t) * (rows * kPTW8 + 8 * 256 * kPTW8 + 8 * 256 + rows) + sizeof(int32_t) * rows +
           sizeof(int16_t) * rows + sizeof(int32_t) * (nleaves + 8);
}

void launch_panel_trsm(cudaStream_t s, const Mat& A, const Mat& Cf, int64_t coef_w0, int nleaves, int64_t tw0,
                       int64_t tw1, const PlsState* st) {
    if (tw1 <= tw0) return;
    const int grid = static_cast<int>((tw1 - tw0 + kPTW8 - 1) / kPTW8);
    k_panel_trsm8<<<grid, 512, panel_trsm8_smem(nleaves), s>>>(A, Cf, coef_w0, nleaves, tw0, tw1, st);
}

// The panel TRSM from a snapshot (look-ahead schedule): the M words come precomputed
// (k_panel_snapshot), so a CTA per leaf j only builds the 8 tables over leaf j's rows
// and adds T[M] to every later row -- no lmap tables or coefficient words per CTA.
// SW = 8: 512-bit strips, a row slice / table entry is 64 B read by 4 lanes (16 B
// each); SW = 1: one word per CTA for the next panel's columns, whose solve is on the
// critical path -- 1/8 of the shared-memory traffic per CTA, so ~8x lower latency.
template <int SW>
__global__ void __launch_bounds__(512, 1)
k_panel_trsm_snap(Mat A, const int64_t* __restrict__ snap, int nleaves, int64_t tw0, int64_t tw1) {
    pdl_wait();
    extern __shared__ __align__(16) uint64_t smem[];
    const int rows_cap = nleaves * 64;
    uint64_t* X = smem;                                               // [rows_cap][SW]
    uint64_t* T = X + rows_cap * SW;                                  // [8][256][SW]
    uint64_t* Mw = T + 8 * 256 * SW;                                  // [rows_cap]
    int16_t* posrow = reinterpret_cast<int16_t*>(Mw + rows_cap);      // [rows_cap]
    int32_t* bstart = reinterpret_cast<int32_t*>(posrow + rows_cap);  // [nleaves + 1]

    const int64_t r0 = snap[0];
    const int nk = static_cast<int>(snap[1]);
    if (nk <= 1) return;
    const int64_t tb = tw0 + static_cast<int64_t>(blockIdx.x) * SW;
    if (tb >= tw1) return;
    const int ntw = static_cast<int>(tw1 - tb < SW ? tw1 - tb : SW);
    const int tid = threadIdx.x;

    for (int i = tid; i < rows_cap; i += 512) posrow[i] = -1;
    for (int j = tid; j <= nleaves; j += 512) bstart[j] = static_cast<int32_t>(snap[kSnapBstart + j]);
    for (int i = tid; i < nk * SW; i += 512) {
        const int t = i / SW, j = i % SW;
        X[i] = j < ntw ? A.w[(r0 + t) * A.stride + tb + j] : 0ull;
    }
    __syncthreads();
    for (int t = tid; t < nk; t += 512) posrow[snap[kSnapQ + t]] = static_cast<int16_t>(t);
    __syncthreads();

    constexpr int kMPer = kMaxTrsmBits / 512;
    uint64_t pf[kMPer];
    auto prefetch = [&](int j) {
        if (j >= nleaves) return;
        const int t0 = bstart[j];
        const int64_t* mj = snap + kSnapM + static_cast<int64_t>(j) * kMaxPanelBits;
#pragma unroll
        for (int u = 0; u < kMPer; ++u) {
            const int t = t0 + tid + u * 512;
            pf[u] = t < nk ? static_cast<uint64_t>(__ldcg(mj + t)) : 0ull;
        }
    };
    prefetch(0);
    for (int j = 0; j < nleaves; ++j) {
        const int t0 = bstart[j], t1 = bstart[j + 1];
        if (t0 == t1) {
            prefetch(j + 1);
            continue;
        }
#pragma unroll
        for (int u = 0; u < kMPer; ++u) {
            const int t = t0 + tid + u * 512;
            if (t < nk) Mw[t] = pf[u];
        }
        prefetch(j + 1);
        if constexpr (SW == 8) {
            // thread = (table g, 16-B chunk wc, low nibble el); high nibble in Gray order
            const int g = tid >> 6, wc = tid & 3, el = (tid >> 2) & 15;
            uint4 v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int l = posrow[64 * j + 8 * g + b];
                v[b] = l >= 0 ? *reinterpret_cast<const uint4*>(X + l * SW + 2 * wc) : make_uint4(0, 0, 0, 0);
            }
            uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((el >> b) & 1) {
                    x.x ^= v[b].x;
                    x.y ^= v[b].y;
                    x.z ^= v[b].z;
                    x.w ^= v[b].w;
                }
            uint64_t* tg = T + g * 256 * SW + 2 * wc;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k) {
                    const uint4 h = v[4 + ((k & 1) ? 0 : ((k & 2) ? 1 : ((k & 4) ? 2 : 3)))];
                    x.x ^= h.x;
                    x.y ^= h.y;
                    x.z ^= h.z;
                    x.w ^= h.w;
                }
                const int eh = k ^ (k >> 1);
                *reinterpret_cast<uint4*>(tg + (eh * 16 + el) * SW) = x;
            }
        } else {
            // thread = (table g, low 6 bits el); the 2 high bits in Gray order
            const int g = tid >> 6, el = tid & 63;
            uint64_t v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int l = posrow[64 * j + 8 * g + b];
                v[b] = l >= 0 ? X[l] : 0ull;
            }
            uint64_t x = 0;
#pragma unroll
            for (int b = 0; b < 6; ++b)
                if ((el >> b) & 1) x ^= v[b];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k) x ^= v[(k & 1) ? 6 : 7];
                const int eh = k ^ (k >> 1);
                T[g * 256 + (eh << 6) + el] = x;
            }
        }
        __syncthreads();
        if constexpr (SW == 8) {
            const int sub = tid & 3, grp = tid >> 2;
            for (int t = t0 + grp; t < nk; t += 128) {
                const uint64_t M = Mw[t];
                uint4 a = *reinterpret_cast<const uint4*>(X + t * SW + 2 * sub);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint4 b =
                        *reinterpret_cast<const uint4*>(T + (g * 256 + ((M >> (8 * g)) & 0xffu)) * SW + 2 * sub);
                    a.x ^= b.x;
                    a.y ^= b.y;
                    a.z ^= b.z;
                    a.w ^= b.w;
                }
                *reinterpret_cast<uint4*>(X + t * SW + 2 * sub) = a;
            }
        } else {
            for (int t = t0 + tid; t < nk; t += 512) {
                const uint64_t M = Mw[t];
                uint64_t a = X[t];
#pragma unroll
                for (int g = 0; g < 8; ++g) a ^= T[g * 256 + ((M >> (8 * g)) & 0xffu)];
                X[t] = a;
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < nk * SW; i += 512) {
        const int t = i / SW, jj = i % SW;
        if (jj < ntw) A.w[(r0 + t) * A.stride + tb + jj] = X[i];
    }
}

template <int SW>
static size_t panel_trsm_snap_smem(int nleaves) {
    const size_t rows = static_cast<size_t>(nleaves) * 64;
    return sizeof(uint64_t) * (rows * SW + 8 * 256 * SW + rows) + sizeof(int16_t) * rows +
           sizeof(int32_t) * (nleaves + 8);
}

void launch_panel_trsm_snap(cudaStream_t s, const Mat& A, const int64_t* snap, int nleaves, int64_t tw0, int64_t tw1,
                            int strip) {
    if (tw1 <= tw0) return;
    if (strip == 1) {
        launch_pdl(k_panel_trsm_snap<1>, dim3(static_cast<unsigned>(tw1 - tw0)), dim3(512),
                   panel_trsm_snap_smem<1>(nleaves), s, A, snap, nleaves, tw0, tw1);
    } else {
        launch_pdl(k_panel_trsm_snap<8>, dim3(static_cast<unsigned>((tw1 - tw0 + 7) / 8)), dim3(512),
                   panel_trsm_snap_smem<8>(nleaves), s, A, snap, nleaves, tw0, tw1);
    }
}

void setup_trsm_kernels() {
    cudaFuncSetAttribute(k_panel_trsm_snap<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(panel_trsm_snap_smem<8>(kMaxTrsmBits / 64)));
    cudaFuncSetAttribute(k_panel_trsm_snap<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(panel_trsm_snap_smem<1>(kMaxTrsmBits / 64)));
    cudaFuncSetAttribute(k_panel_trsm8, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(panel_trsm8_smem(kMaxTrsmBits / 64)));
    cudaFuncSetAttribute(k_pivot_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(trsm_smem(kMaxTrsmBits / 64)));
}

}  // namespace f2g
