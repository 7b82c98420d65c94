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

namespace f2g {

namespace {

constexpr int kThreads = 512;
constexpr int kRPT = 4;
constexpr int kTM = (kThreads / 32) * 4 * kRPT;  // 256 rows per CTA (fills all SMs at m = 64K)
constexpr int kTNW = 16;                         // 1024-bit column tile
// smem: X[64][kTNW] | T[2][256][kTNW] | F[8][256] | cbuf[kTM] | pbuf[kTM]
constexpr size_t kSmem = sizeof(uint64_t) * (64 * kTNW + 2 * 256 * kTNW + 8 * 256 + 2 * kTM);

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 2)
k_leaf_update(Mat A, int64_t wl, int64_t rw0, int64_t rw1, const int64_t* pmap, const PlsState* st) {
    __shared__ uint64_t suf[64];
    __shared__ int sq[64];
    __shared__ int gstart[9];
    __shared__ int16_t posrow[64];
    __shared__ uint8_t Ms[8 * 256];
    extern __shared__ __align__(16) uint64_t dsm[];
    uint64_t* X = dsm;                                        // [64][kTNW]
    uint64_t* Tb = X + 64 * kTNW;                             // [2][256][kTNW]
    uint64_t* F = Tb + 2 * 256 * kTNW;                        // [8][256] finalize corrections
    uint64_t* cbuf = F + 8 * 256;                             // [kTM]
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

    // tables prepared by k_leaf_pivot (depend only on the leaf's pivots)
    for (int i = tid; i < 8 * 256; i += kThreads) F[i] = (&st->leaf_F[0][0])[i];
    for (int i = tid; i < 8 * 256 / 4; i += kThreads)
        reinterpret_cast<uint32_t*>(Ms)[i] = reinterpret_cast<const uint32_t*>(&st->leaf_M[0][0])[i];
    if (tid < 64) {
        suf[tid] = st->ufull[tid];
        sq[tid] = st->q[tid];
        posrow[tid] = -1;
    }
    __syncthreads();
    if (tid < kb) posrow[sq[tid]] = static_cast<int16_t>(tid);
    if (tid <= 8) {
        int lo = 0;
        while (lo < kb && sq[lo] < 8 * tid) ++lo;
        gstart[tid] = lo;
    }

    // 1. finalise the leaf word of the tile's rows -> coefficient words
    for (int i = tid; i < nrows; i += kThreads) {
        const int64_t phys = pmap[row_base + i];
        uint64_t w = A.w[phys * A.stride + wl];
#pragma unroll
        for (int g = 0; g < 8; ++g) w ^= F[g * 256 + ((w >> (8 * g)) & 0xffu)];
        cbuf[i] = w;
        pbuf[i] = phys;
        if (blockIdx.x == 0) A.w[phys * A.stride + wl] = w;
    }
    if (ntw == 0) return;

    // pivot rows' slice of the tile
    for (int i = tid; i < kb * kTNW; i += kThreads) {
        const int t = i / kTNW, k = i % kTNW;
        X[i] = k < ntw ? A.w[pmap[r0 + t] * A.stride + tile_w0 + k] : 0ull;
    }
    __syncthreads();

    const int rq = lane >> 3, wp = lane & 7;
    uint64_t acc0[kRPT], acc1[kRPT];
#pragma unroll
    for (int j = 0; j < kRPT; ++j) {
        const int i = warp * 4 * kRPT + rq + 4 * j;
        acc0[j] = acc1[j] = 0;
        if (i < nrows) {
            const uint64_t* cr = A.w + pbuf[i] * A.stride + tile_w0;
            if (2 * wp < ntw) acc0[j] = cr[2 * wp];
            if (2 * wp + 1 < ntw) acc1[j] = cr[2 * wp + 1];
        }
    }

    // 2./3. per group of 8 leaf columns: a table T over the group's pivot rows as they
    // are now; the group's pivot rows and every later row add T[M(c)] (c = the row's
    // coefficient byte, masked below its own pivot for the group's rows), which
    // equals adding the combination of the *solved* group rows (see trsm.cu)
    for (int g = 0; g < 8; ++g) {
        const int g0 = gstart[g], g1 = gstart[g + 1];
        if (g0 == g1) continue;
        const int sh = 8 * g;
        const uint8_t* Mg = Ms + g * 256;
        uint64_t* tb = Tb + (g & 1) * 256 * kTNW;
        // table: 4 warps, thread = (16-byte column chunk wp, low nibble el), Gray walk
        if (warp < 4) {
            const int el = tid >> 3;  // 0..15
            uint64_t v0[8], v1[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int r = posrow[sh + b];
                v0[b] = r >= 0 ? X[r * kTNW + 2 * wp] : 0ull;
                v1[b] = r >= 0 ? X[r * kTNW + 2 * wp + 1] : 0ull;
            }
            uint64_t l0 = 0, l1 = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((el >> b) & 1) {
                    l0 ^= v0[b];
                    l1 ^= v1[b];
                }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k) {
                    const int b = 4 + ((k & 1) ? 0 : ((k & 2) ? 1 : ((k & 4) ? 2 : 3)));
                    l0 ^= v0[b];
                    l1 ^= v1[b];
                }
                const int eh = k ^ (k >> 1);
                uint64_t* e = tb + (eh * 16 + el) * kTNW + 2 * wp;
                e[0] = l0;
                e[1] = l1;
            }
        }
        __syncthreads();
        for (int i = tid; i < (kb - g0) * kTNW; i += kThreads) {
            const int t = g0 + i / kTNW, k = i % kTNW;
            uint32_t cb = static_cast<uint32_t>(suf[t] >> sh) & 0xffu;
            if (t < g1) cb &= (1u << (sq[t] - sh)) - 1u;
            X[t * kTNW + k] ^= tb[Mg[cb] * kTNW + k];
        }
#pragma unroll
        for (int j = 0; j < kRPT; ++j) {
            const int i = warp * 4 * kRPT + rq + 4 * j;
            const unsigned idx = Mg[static_cast<unsigned>(cbuf[i] >> sh) & 0xffu];
            const uint4 v = lds128(tb + idx * kTNW + 2 * wp);
            acc0[j] ^= static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32);
            acc1[j] ^= static_cast<uint64_t>(v.z) | (static_cast<uint64_t>(v.w) << 32);
        }
        __syncthreads();
    }

#pragma unroll
    for (int j = 0; j < kRPT; ++j) {
        const int i = warp * 4 * kRPT + rq + 4 * j;
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
