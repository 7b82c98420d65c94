// One leaf's update of the rest of its panel (k_leaf_update).
//
// After k_leaf_pivot has found the leaf's kb pivots (positions leaf_r..leaf_r+kb,
// their final leaf words in st->ufull, strict parts in st->ustrict), this kernel
//   1. finalises the leaf word of every row below the pivots: the elimination
//      chain of gauss_pls (proj/src/gauss.cpp:47-49) restricted to the leaf word,
//      which leaves exactly the row's L coefficients at the pivot columns.  The
//      chain runs 8 pivot columns at a time through 256-entry correction tables
//      (the corrected-prefix idea of make_table1, proj/src/mmpf.cpp:54-77) that
//      k_leaf_pivot prepares once per leaf;
//   2. solves the pivot rows over the panel columns right of the leaf
//      (U = L11^{-1} A12, trsm_lower_left_unit, mul.cpp:109-131), 8 pivot columns
//      at a time;
//   3. adds into every other row, per 8 coefficient bits, one row of the 256-entry
//      table of combinations of the solved pivot rows (add_rows_from_table,
//      m4ri.cpp:28-38).
// The table of group g serves both the later pivot rows (step 2) and all other
// rows (step 3), so each is built once per CTA.  Rows are addressed through pmap
// (the panel's virtual row order).  Grid: x = 1024-bit column tiles of the panel
// remainder (one empty tile when the leaf ends the panel), y = 1024-row tiles.
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"
#include "leafupd_body.cuh"

namespace f2g {

namespace {
constexpr int kThreads = 512;
constexpr int kTM = (kThreads / 32) * 4 * kLuRPT;  // 256 rows per CTA (fills all SMs at m = 64K)
constexpr int kTNW = kLuTNW;
}  // namespace

__global__ void __launch_bounds__(kThreads, 2)
k_leaf_update(Mat A, int64_t wl, int64_t rw0, int64_t rw1, const int64_t* pmap, const PlsState* st) {
    extern __shared__ __align__(16) uint64_t dsm[];
    leaf_update_body<kThreads>(A, wl, rw0, rw1, pmap, st, blockIdx.x, blockIdx.y, dsm);
}

void launch_leaf_update(cudaStream_t s, const Mat& A, int64_t wl, int64_t rw0, int64_t rw1, const int64_t* pmap,
                        const PlsState* st) {
    const int gx = rw1 > rw0 ? static_cast<int>((rw1 - rw0 + kTNW - 1) / kTNW) : 1;
    const int gy = static_cast<int>((A.m + kTM - 1) / kTM);
    k_leaf_update<<<dim3(gx, gy < 1 ? 1 : gy), kThreads, leaf_update_smem(kThreads), s>>>(A, wl, rw0, rw1, pmap, st);
}

void setup_leafupd_kernels() {
    cudaFuncSetAttribute(k_leaf_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(leaf_update_smem(kThreads)));
}

}  // namespace f2g
