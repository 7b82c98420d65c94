// Pivot-row triangular solve over GF(2).
//
// X_t = B_t xor sum_{l<t} L[t][l] X_l for the kb pivot rows of a leaf/panel
// (or an explicit unit-lower L), i.e. B <- L^{-1} B as trsm_lower_left_unit
// does (proj/src/mul.cpp:109-131; the diagonal is implicit and everything on
// or above it ignored).  L is read in "raw" form: row t's coefficient for
// pivot l sits at the pivot's raw column q_l of its coefficient words, which
// is how the packed layout stores L before compress_columns (gauss.cpp:47-53).
//
// Blocking: each CTA owns TW target words of all kb rows in SMEM and walks the
// raw columns 8 at a time.  For each group it solves the (<= 8) pivots inside
// the group, builds the 256-entry Gray table of their combinations, and adds
// one table row into every later pivot row (one lookup per row per group).
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kTW = 8;           // target words per CTA
constexpr int kMaxRows = kMaxPanelBits;

struct TrsmCtx {
    int64_t kb, r0;
    const int32_t* q;  // nullptr => identity pivots
};

}  // namespace

__global__ void __launch_bounds__(256)
k_pivot_trsm(Mat A, int64_t coef_w0, int coef_words, int64_t tw0, int64_t tw1, const PlsState* st,
             PivotSet ps, Mat L) {
    extern __shared__ __align__(16) uint64_t smem[];
    uint64_t* X = smem;                          // [kMaxRows][kTW]
    uint64_t* T = X + kMaxRows * kTW;            // [256][kTW]
    uint64_t* cw = T + 256 * kTW;                // [kMaxRows] coefficient word of the current 8 groups
    int32_t* sq = reinterpret_cast<int32_t*>(cw + kMaxRows);  // [kMaxRows]
    int32_t* gstart = sq + kMaxRows;             // [kMaxPanelBits/8 + 1]

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

    for (int t = tid; t < nk; t += nth) sq[t] = qsrc ? qsrc[t] : t;
    for (int i = tid; i < nk * kTW; i += nth) {
        int t = i / kTW, j = i % kTW;
        X[i] = j < ntw ? A.w[(r0 + t) * A.stride + tb + j] : 0ull;
    }
    __syncthreads();
    const int ngroups = coef_words * 8;
    for (int g = tid; g <= ngroups; g += nth) {
        int lo = 0, hi = nk;  // first t with sq[t] >= 8g
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (sq[mid] < 8 * g) lo = mid + 1;
            else hi = mid;
        }
        gstart[g] = lo;
    }

    for (int g = 0; g < ngroups; ++g) {
        if ((g & 7) == 0) {
            // stage coefficient word g/8 of every pivot row
            __syncthreads();
            for (int t = tid; t < nk; t += nth)
                cw[t] = ps.mode == 2 ? L.w[static_cast<int64_t>(t) * L.stride + (g >> 3)]
                                     : A.w[(r0 + t) * A.stride + coef_w0 + (g >> 3)];
        }
        __syncthreads();
        const int t0 = gstart[g], t1 = gstart[g + 1];
        if (t0 == t1) continue;
        const int sh = 8 * (g & 7), base = 8 * g;
        if (t1 - t0 > 1 && tid < kTW) {
            // in-group forward substitution, rows held in registers
            const int j = tid, ng = t1 - t0;
            uint64_t x[8];
            int qb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x[u] = u < ng ? X[(t0 + u) * kTW + j] : 0ull;
                qb[u] = u < ng ? sq[t0 + u] - base : 8;
            }
#pragma unroll
            for (int u = 1; u < 8; ++u) {
                if (u < ng) {
                    const unsigned cb = static_cast<unsigned>(cw[t0 + u] >> sh) & 0xffu;
#pragma unroll
                    for (int l = 0; l < u; ++l)
                        if ((cb >> qb[l]) & 1u) x[u] ^= x[l];
                }
            }
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u < ng) X[(t0 + u) * kTW + j] = x[u];
        }
        if (t1 >= nk) break;
        __syncthreads();
        // table of the group's solved rows: thread = (target word j, low nibble el),
        // high nibble walked in Gray order (one XOR per entry)
        if (tid < kTW * 16) {
            const int j = tid % kTW, el = tid / kTW;
            uint64_t v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) v[b] = 0;
            for (int l = t0; l < t1; ++l) {
                const int b = sq[l] - base;
#pragma unroll
                for (int bb = 0; bb < 8; ++bb)
                    if (bb == b) v[bb] = X[l * kTW + j];
            }
            uint64_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((el >> b) & 1) x ^= v[b];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k) x ^= v[4 + ((k & 1) ? 0 : ((k & 2) ? 1 : ((k & 4) ? 2 : 3)))];
                const int eh = k ^ (k >> 1);
                T[(eh * 16 + el) * kTW + j] = x;
            }
        }
        __syncthreads();
        for (int t = t1 + tid; t < nk; t += nth) {
            const unsigned cb = static_cast<unsigned>(cw[t] >> sh) & 0xffu;
            uint4* xr = reinterpret_cast<uint4*>(X + t * kTW);
            const uint4* tr = reinterpret_cast<const uint4*>(T + cb * kTW);
#pragma unroll
            for (int j = 0; j < kTW / 2; ++j) {
                uint4 a = xr[j];
                const uint4 b = tr[j];
                a.x ^= b.x;
                a.y ^= b.y;
                a.z ^= b.z;
                a.w ^= b.w;
                xr[j] = a;
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < nk * kTW; i += nth) {
        int t = i / kTW, j = i % kTW;
        if (j < ntw) A.w[(r0 + t) * A.stride + tb + j] = X[i];
    }
}

static size_t trsm_smem() {
    return sizeof(uint64_t) * (kMaxRows * kTW + 256 * kTW + kMaxRows) + sizeof(int32_t) * (kMaxRows + kMaxPanelBits / 8 + 8);
}

void launch_pivot_trsm(cudaStream_t s, const Mat& A, int64_t coef_w0, int coef_words, int64_t tw0,
                       int64_t tw1, const PlsState* st, PivotSet ps, const Mat* L) {
    if (tw1 <= tw0) return;
    const int grid = static_cast<int>((tw1 - tw0 + kTW - 1) / kTW);
    Mat l = L ? *L : Mat{nullptr, 0, 0, 0};
    k_pivot_trsm<<<grid, 256, trsm_smem(), s>>>(A, coef_w0, coef_words, tw0, tw1, st, ps, l);
}

void setup_trsm_kernels() {
    cudaFuncSetAttribute(k_pivot_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(trsm_smem()));
}

}  // namespace f2g
