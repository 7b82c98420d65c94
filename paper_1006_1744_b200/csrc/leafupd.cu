// One leaf's update of the rest of its panel (k_leaf_update).
//
// After k_leaf_pivot has found the leaf's kb pivots (positions leaf_r..leaf_r+kb,
// their final leaf words in st->ufull, strict parts in st->ustrict), this kernel
//   1. finalises the leaf word of every row below the pivots: the elimination
//      chain of gauss_pls (proj/src/gauss.cpp:47-49) restricted to the leaf word,
//      which leaves exactly the row's L coefficients at the pivot columns;
//   2. solves the pivot rows over the panel columns right of the leaf
//      (U = L11^{-1} A12, trsm_lower_left_unit, mul.cpp:109-131), 8 pivot columns
//      at a time;
//   3. adds into every other row, per 8 coefficient bits, one row of the 256-entry
//      table of combinations of the solved pivot rows (add_rows_from_table,
//      m4ri.cpp:28-38, with make_table1's corrected ids, mmpf.cpp:54-77: the
//      coefficient byte already is the combination, so no id fix-up is needed).
// The table of group g serves both the later pivot rows (step 2) and all other
// rows (step 3), so each is built once per CTA.  Rows are addressed through pmap
// (the panel's virtual row order).  Grid: x = 512-bit column tiles of the panel
// remainder (one empty tile when the leaf ends the panel), y = 1024-row tiles.
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kThreads = 512;
constexpr int kRPT = 8;
constexpr int kTM = (kThreads / 32) * 8 * kRPT;  // 1024 rows per CTA
constexpr int kTNW = 8;                          // 512-bit column tile
constexpr size_t kSmem = sizeof(uint64_t) * (64 * kTNW + 2 * 256 * kTNW + 2 * kTM);

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
k_leaf_update(Mat A, int64_t wl, int64_t rw0, int64_t rw1, const int64_t* pmap, const PlsState* st) {
    __shared__ uint64_t su[64], suf[64];
    __shared__ int sq[64];
    __shared__ int gstart[9];
    extern __shared__ __align__(16) uint64_t dsm[];
    uint64_t* X = dsm;                                        // [64][kTNW]
    uint64_t* Tb = X + 64 * kTNW;                             // [2][256][kTNW]
    uint64_t* cbuf = Tb + 2 * 256 * kTNW;                     // [kTM]
    int64_t* pbuf = reinterpret_cast<int64_t*>(cbuf + kTM);   // [kTM]

    const int kb = static_cast<int>(st->leaf_kb);
    if (kb == 0) return;
    const int64_t r0 = st->leaf_r;
    const int64_t row_base = r0 + kb + static_cast<int64_t>(blockIdx.y) * kTM;
    if (row_base >= A.m && blockIdx.y != 0) return;
    const int64_t nrows64 = A.m - row_base;
    const int nrows = nrows64 <= 0 ? 0 : (nrows64 < kTM ? static_cast<int>(nrows64) : kTM);
    const int64_t tile_w0 = rw0 + static_cast<int64_t>(blockIdx.x) * kTNW;
    const int ntw = tile_w0 >= rw1 ? 0 : static_cast<int>(rw1 - tile_w0 < kTNW ? rw1 - tile_w0 : kTNW);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid < 64) {
        su[tid] = st->ustrict[tid];
        suf[tid] = st->ufull[tid];
        sq[tid] = st->q[tid];
    }
    __syncthreads();

    // 1. finalise the leaf word of the tile's rows -> coefficient words
    for (int i = tid; i < nrows; i += kThreads) {
        const int64_t phys = pmap[row_base + i];
        uint64_t w = A.w[phys * A.stride + wl];
        for (int l = 0; l < kb; ++l)
            if ((w >> sq[l]) & 1ull) w ^= su[l];
        cbuf[i] = w;
        pbuf[i] = phys;
        if (blockIdx.x == 0) A.w[phys * A.stride + wl] = w;
    }
    if (ntw == 0) return;

    // pivot rows' slice of the tile, and the 8-column groups of pivots
    for (int i = tid; i < kb * kTNW; i += kThreads) {
        const int t = i / kTNW, k = i % kTNW;
        X[i] = k < ntw ? A.w[pmap[r0 + t] * A.stride + tile_w0 + k] : 0ull;
    }
    if (tid <= 8) {
        int lo = 0;
        while (lo < kb && sq[lo] < 8 * tid) ++lo;
        gstart[tid] = lo;
    }
    __syncthreads();

    const int rq = lane >> 2, wp = lane & 3;
    uint64_t acc0[kRPT], acc1[kRPT];
#pragma unroll
    for (int j = 0; j < kRPT; ++j) {
        const int i = warp * 64 + rq + 8 * j;
        acc0[j] = acc1[j] = 0;
        if (i < nrows) {
            const uint64_t* cr = A.w + pbuf[i] * A.stride + tile_w0;
            if (2 * wp < ntw) acc0[j] = cr[2 * wp];
            if (2 * wp + 1 < ntw) acc1[j] = cr[2 * wp + 1];
        }
    }

    for (int g = 0; g < 8; ++g) {
        const int g0 = gstart[g], g1 = gstart[g + 1];
        if (g0 == g1) continue;
        const int sh = 8 * g;
        // (a) pivots inside the group, in registers (one thread per tile word)
        if (tid < kTNW && g1 - g0 > 1) {
            const int k = tid, ng = g1 - g0;
            uint64_t x[8];
            int qb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x[u] = u < ng ? X[(g0 + u) * kTNW + k] : 0ull;
                qb[u] = u < ng ? sq[g0 + u] - sh : 8;
            }
#pragma unroll
            for (int u = 1; u < 8; ++u) {
                if (u < ng) {
                    const unsigned cb = static_cast<unsigned>(suf[g0 + u] >> sh) & ((1u << qb[u]) - 1u);
#pragma unroll
                    for (int l = 0; l < u; ++l)
                        if ((cb >> qb[l]) & 1u) x[u] ^= x[l];
                }
            }
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u < ng) X[(g0 + u) * kTNW + k] = x[u];
        }
        __syncthreads();
        // (b) table of the group's solved rows, indexed by the raw coefficient byte
        uint64_t* tb = Tb + (g & 1) * 256 * kTNW;
        for (int i = tid; i < 256 * kTNW; i += kThreads) {
            const int e = i / kTNW, k = i % kTNW;
            uint64_t v = 0;
            for (int l = g0; l < g1; ++l)
                if ((e >> (sq[l] - sh)) & 1) v ^= X[l * kTNW + k];
            tb[i] = v;
        }
        __syncthreads();
        // (c) later pivot rows and all other rows add one table row each
        for (int i = tid; i < (kb - g1) * kTNW; i += kThreads) {
            const int t = g1 + i / kTNW, k = i % kTNW;
            X[t * kTNW + k] ^= tb[((suf[t] >> sh) & 0xffu) * kTNW + k];
        }
#pragma unroll
        for (int j = 0; j < kRPT; ++j) {
            const int i = warp * 64 + rq + 8 * j;
            const unsigned idx = static_cast<unsigned>(cbuf[i < kTM ? i : 0] >> sh) & 0xffu;
            const uint4 v = lds128(tb + idx * kTNW + 2 * wp);
            acc0[j] ^= static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32);
            acc1[j] ^= static_cast<uint64_t>(v.z) | (static_cast<uint64_t>(v.w) << 32);
        }
        __syncthreads();
    }

#pragma unroll
    for (int j = 0; j < kRPT; ++j) {
        const int i = warp * 64 + rq + 8 * j;
        if (i < nrows) {
            uint64_t* cr = A.w + pbuf[i] * A.stride + tile_w0;
            if (2 * wp < ntw) cr[2 * wp] = acc0[j];
            if (2 * wp + 1 < ntw) cr[2 * wp + 1] = acc1[j];
        }
    }
    if (blockIdx.y == 0)
        for (int i = tid; i < kb * kTNW; i += kThreads) {
            const int t = i / kTNW, k = i % kTNW;
            if (k < ntw) A.w[pmap[r0 + t] * A.stride + tile_w0 + k] = X[i];
        }
}

void launch_leaf_update(cudaStream_t s, const Mat& A, int64_t wl, int64_t rw0, int64_t rw1, const int64_t* pmap,
                        const PlsState* st) {
    const int gx = rw1 > rw0 ? static_cast<int>((rw1 - rw0 + kTNW - 1) / kTNW) : 1;
    const int gy = static_cast<int>((A.m + kTM - 1) / kTM);
    k_leaf_update<<<dim3(gx, gy < 1 ? 1 : gy), kThreads, kSmem, s>>>(A, wl, rw0, rw1, pmap, st);
}

void setup_leafupd_kernels() {
    cudaFuncSetAttribute(k_leaf_update, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
}

}  // namespace f2g
