// Panel bookkeeping kernels of the PLS engine (the pivot search itself is the
// panel kernel, panel.cu):
//
//   k_perm_save/put at the end of a panel, the panel's transpositions (which the
//                   leaves only recorded as a re-mapped virtual row order, pmap)
//                   applied to whole rows in one gather
//   k_panel_lmaps   per-leaf L11^{-1} byte maps rebuilt from a panel's words (a
//                   rank that imports a panel factored elsewhere)
//   k_dist_*        the column-sharded exchange (export / import of a panel)
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
// Exchange buffer of one panel (api.cu, f2_dist_*): the panel's words of row x at
// [x * ws, (x+1) * ws), then the header at m * ws (int64): [0] kb, [1] panel_r,
// [2] nmoved, [3] the panel's global first column, [4, 4+W) pivot columns (panel
// relative), [4+W, 4+2W) P entries P[panel_r + t], then kMaxMoved re-mapped
// positions and kMaxMoved source rows (pmap values).
__global__ void __launch_bounds__(256) k_dist_export(const PlsState* st, const int64_t* pmap, const int64_t* P,
                                                    int64_t* hdr, int W, int64_t col) {
    const int kb = static_cast<int>(st->panel_kb), nm = st->nmoved;
    const int64_t r0 = st->panel_r;
    int64_t* q = hdr + 4;
    int64_t* pp = q + W;
    int64_t* mv = pp + W;
    int64_t* src = mv + kMaxMoved;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    if (tid == 0) {
        hdr[0] = kb;
        hdr[1] = r0;
        hdr[2] = nm;
        hdr[3] = col;
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

// The owner's panel words of every row >= panel_r, in the row order the panel's
// gather will produce (position x reads physical row pmap[x]), so the broadcast can
// leave before the owner's own gather runs; words past the panel's width are zero.
__global__ void __launch_bounds__(256) k_dist_export_words(Mat A, int64_t pw0, int nwp, const PlsState* st,
                                                          const int64_t* pmap, uint64_t* buf, int ws) {
    const int64_t r0 = st->panel_r;
    const int per = ws / 2;  // 16-byte chunks per row (ws is even: W is a multiple of 128)
    const int64_t total = (A.m - r0) * per;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t x = r0 + i / per;
        const int k = 2 * static_cast<int>(i % per);
        const int64_t ph = pmap[x];
        uint4 v = make_uint4(0, 0, 0, 0);
        if (k + 1 < nwp) {
            v = *reinterpret_cast<const uint4*>(A.w + ph * A.stride + pw0 + k);
        } else if (k < nwp) {
            const uint64_t w = A.w[ph * A.stride + pw0 + k];
            v.x = static_cast<unsigned>(w);
            v.y = static_cast<unsigned>(w >> 32);
        }
        *reinterpret_cast<uint4*>(buf + x * ws + k) = v;
    }
}

// A rank that does not own the panel adopts the owner's header: pivot bookkeeping
// for the TRSM/Schur kernels, P and the pivot columns, and the re-mapped positions
// for the row gather.
__global__ void __launch_bounds__(1024) k_dist_import(PlsState* st, int64_t* pmap, int64_t* P, int64_t* Qp,
                                                     const int64_t* hdr, int W) {
    const int kb = static_cast<int>(hdr[0]), nm = static_cast<int>(hdr[2]);
    const int64_t r0 = hdr[1], col = hdr[3];
    const int64_t* q = hdr + 4;
    const int64_t* pp = q + W;
    const int64_t* mv = pp + W;
    const int64_t* src = mv + kMaxMoved;
    const int tid = threadIdx.x, nth = blockDim.x;
    for (int i = tid; i < W; i += nth) st->brow[i] = -1;
    __syncthreads();
    for (int t = tid; t < kb; t += nth) {
        st->panel_q[t] = static_cast<int32_t>(q[t]);
        st->brow[q[t]] = r0 + t;
        P[r0 + t] = pp[t];
        Qp[r0 + t] = col + q[t];
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

void launch_dist_export(cudaStream_t s, const Mat& A, int64_t pw0, int nwp, const PlsState* st, const int64_t* pmap,
                        const int64_t* P, uint64_t* buf, int W, int64_t col, int nsm) {
    const int ws = W / 64;
    k_dist_export_words<<<nsm * 4, 256, 0, s>>>(A, pw0, nwp, st, pmap, buf, ws);
    k_dist_export<<<32, 256, 0, s>>>(st, pmap, P, reinterpret_cast<int64_t*>(buf + A.m * ws), W, col);
}
void launch_dist_import(cudaStream_t s, PlsState* st, int64_t* pmap, int64_t* P, int64_t* Qp, const int64_t* hdr,
                        int W) {
    k_dist_import<<<1, 1024, 0, s>>>(st, pmap, P, Qp, hdr, W);
}

// Snapshot of a finished panel (see kernels.cuh, kSnap*): block (j, y) handles leaf j's
// solve words of pivots t = 256 y + tid.  The pivot rows' coefficient words are read
// from Cf at position panel_r + t, through rowmap when the panel's row gather has not
// run yet (the virtual order: physical row rowmap[x]).
__device__ __forceinline__ void snapshot_block(const PlsState* st, int64_t* snap, const Mat& Cf, int64_t coef_w0,
                                               int nleaves, int j, int by, const int64_t* rowmap) {
    __shared__ int s_b[2];
    const int tid = threadIdx.x;
    const int t = by * 256 + tid;
    const int64_t r0 = st->panel_r;
    const int nk = static_cast<int>(st->panel_kb);
    const int pb = nleaves * 64;
    auto lower = [&](int v) {  // first pivot index with column >= v (panel_q ascends)
        int lo = 0, hi = nk;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (st->panel_q[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    if (tid < 2) s_b[tid] = lower(64 * (j + tid));
    if (j == 0 && t < pb) {
        if (t == 0) {
            snap[0] = r0;
            snap[1] = nk;
        }
        snap[kSnapBrow + t] = st->brow[t];
        snap[kSnapQ + t] = t < nk ? st->panel_q[t] : -1;
        if (t <= nleaves) snap[kSnapBstart + t] = lower(64 * t);
    }
    __syncthreads();
    const int t0 = s_b[0], t1 = s_b[1];
    if (t >= t0 && t < nk) {
        const int64_t row = rowmap ? rowmap[r0 + t] : r0 + t;
        uint64_t c = Cf.w[row * Cf.stride + coef_w0 + j];
        if (t < t1) c &= (1ull << (st->panel_q[t] - 64 * j)) - 1ull;
        uint64_t M = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) M ^= st->lmap[j][g][(c >> (8 * g)) & 0xffu];
        snap[kSnapM + static_cast<int64_t>(j) * kMaxPanelBits + t] = static_cast<int64_t>(M);
    }
}

// Panel end, step 1: copy the rows that the panel's positions now refer to
// (physical row pmap[x] for every re-mapped position x) into scratch, whole width.
// Blocks past the copy (when snap != nullptr) take the panel's snapshot meanwhile,
// reading the pivot rows through pmap: one launch instead of two on the serial path.
__global__ void __launch_bounds__(256) k_perm_save(Mat A, int64_t nwords, const PlsState* st, const int64_t* pmap,
                                                  uint64_t* scratch, unsigned gx, unsigned gy, int64_t* snap, Mat Cf,
                                                  int64_t coef_w0, int nleaves, int64_t* plan) {
    pdl_wait();
    const unsigned b = blockIdx.x;
    if (b >= gx * gy) {
        const unsigned s = b - gx * gy;
        snapshot_block(st, snap, Cf, coef_w0, nleaves, static_cast<int>(s % nleaves), static_cast<int>(s / nleaves),
                       Cf.w == A.w ? pmap : nullptr);
        return;
    }
    const int n = st->nmoved;
    if (plan && b == 0) {  // the gather as (destination, source) row pairs, for k_plan_save/put
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t x = st->moved[i];
            plan[1 + 2 * i] = x;
            plan[2 + 2 * i] = pmap[x];
        }
        if (threadIdx.x == 0) plan[0] = n;
    }
    const int64_t k = 2 * (static_cast<int64_t>(b % gx) * blockDim.x + threadIdx.x);  // word pair (16 B)
    if (k >= nwords) return;
    for (int i = b / gx; i < n; i += gy) {
        const uint64_t* src = A.w + pmap[st->moved[i]] * A.stride + k;
        uint64_t* dst = scratch + static_cast<int64_t>(i) * A.stride + k;
        if (k + 1 < nwords) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
        else dst[0] = src[0];
    }
}

// Panel end, step 2: physical row x <- saved content, pmap back to identity.
// This applies the panel's transpositions (perm.cpp:8-16) to every column.
__global__ void __launch_bounds__(256) k_perm_put(Mat A, int64_t nwords, const PlsState* st, int64_t* pmap,
                                                 const uint64_t* scratch) {
    pdl_wait();
    const int n = st->nmoved;
    const int64_t k = 2 * (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
    for (int i = blockIdx.y; i < n; i += gridDim.y) {
        const int64_t x = st->moved[i];
        const uint64_t* src = scratch + static_cast<int64_t>(i) * A.stride + k;
        uint64_t* dst = A.w + x * A.stride + k;
        if (k + 1 < nwords) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
        else if (k < nwords) dst[0] = src[0];
        if (k == 0) pmap[x] = x;
    }
}

// The same gather on words [w0, w1) only, from a plan k_perm_save recorded: the columns
// a streamed upload delivers after the panel's own gather ran (api.cu, enqueue_engine).
__global__ void __launch_bounds__(256) k_plan_save(Mat A, int64_t w0, int64_t w1, const int64_t* plan,
                                                  uint64_t* scratch, unsigned gx, unsigned gy) {
    const int n = static_cast<int>(plan[0]);
    const int64_t k = w0 + 2 * (static_cast<int64_t>(blockIdx.x % gx) * blockDim.x + threadIdx.x);
    if (k >= w1) return;
    for (int i = blockIdx.x / gx; i < n; i += gy) {
        const uint64_t* src = A.w + plan[2 + 2 * i] * A.stride + k;
        uint64_t* dst = scratch + static_cast<int64_t>(i) * A.stride + k;
        if (k + 1 < w1) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
        else dst[0] = src[0];
    }
}

__global__ void __launch_bounds__(256) k_plan_put(Mat A, int64_t w0, int64_t w1, const int64_t* plan,
                                                 const uint64_t* scratch, unsigned gx, unsigned gy) {
    const int n = static_cast<int>(plan[0]);
    const int64_t k = w0 + 2 * (static_cast<int64_t>(blockIdx.x % gx) * blockDim.x + threadIdx.x);
    if (k >= w1) return;
    for (int i = blockIdx.x / gx; i < n; i += gy) {
        const uint64_t* src = scratch + static_cast<int64_t>(i) * A.stride + k;
        uint64_t* dst = A.w + plan[1 + 2 * i] * A.stride + k;
        if (k + 1 < w1) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
        else dst[0] = src[0];
    }
}

__global__ void k_pmap_init(int64_t* pmap, int64_t m) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        pmap[i] = i;
}


void launch_perm(cudaStream_t s, const Mat& A, int64_t nwords, const PlsState* st, int64_t* pmap, uint64_t* scratch,
                 int64_t* snap, int nleaves, const Mat* Cf, int64_t coef_w0, int64_t* plan) {
    // rows are 128-byte aligned (stride % 16 words == 0): 16-byte accesses, ~1024 CTAs
    const unsigned gx = static_cast<unsigned>((nwords + 511) / 512);
    const unsigned gy = gx >= 1024 ? 1u : 1024u / gx;
    const unsigned nsnap = snap ? static_cast<unsigned>(nleaves * ((nleaves * 64 + 255) / 256)) : 0u;
    const Mat cf = Cf ? *Cf : A;
    launch_pdl(k_perm_save, dim3(gx * gy + nsnap), dim3(256), 0, s, A, nwords, st, static_cast<const int64_t*>(pmap),
               scratch, gx, gy, snap, cf, coef_w0, nleaves, plan);
    launch_pdl(k_perm_put, dim3(gx, gy), dim3(256), 0, s, A, nwords, st, pmap, static_cast<const uint64_t*>(scratch));
}

void launch_plan_perm(cudaStream_t s, const Mat& A, int64_t w0, int64_t w1, const int64_t* plan, uint64_t* scratch) {
    if (w1 <= w0) return;
    const unsigned gx = static_cast<unsigned>((w1 - w0 + 511) / 512);
    const unsigned gy = gx >= 1024 ? 1u : 1024u / gx;
    k_plan_save<<<gx * gy, 256, 0, s>>>(A, w0, w1, plan, scratch, gx, gy);
    k_plan_put<<<gx * gy, 256, 0, s>>>(A, w0, w1, plan, static_cast<const uint64_t*>(scratch), gx, gy);
}

void launch_pmap_init(cudaStream_t s, int64_t* pmap, int64_t m) {
    int64_t g = (m + 255) / 256;
    if (g > 1024) g = 1024;
    if (g < 1) g = 1;
    k_pmap_init<<<static_cast<int>(g), 256, 0, s>>>(pmap, m);
}

void setup_leaf_kernels() {}

}  // namespace f2g
