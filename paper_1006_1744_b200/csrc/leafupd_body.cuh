// Device body of the leaf update, shared by k_leaf_update (leafupd.cu) and the
// persistent panel kernel (panel.cu).  See leafupd.cu for the algorithm.
#pragma once
#include <cstdint>

#include "f2gpu.cuh"

namespace f2g {

namespace lu {


__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

}  // namespace lu

// Row tile `ty` (kTM = NT/8 * kRPT rows from leaf_r + kb), column tile `tx` of the
// panel remainder.  All loads of matrix words, pmap and the state go through L2:
// the persistent panel kernel runs this right after other CTAs wrote them.
template <int NT>
static __device__ __noinline__ void leaf_update_body(const Mat& A, int64_t wl, int64_t rw0, int64_t rw1, const int64_t* pmap,
                                 const PlsState* st, int tx, int ty, uint64_t* dsm) {
    constexpr int kTM = (NT / 32) * 4 * kLuRPT;
    constexpr int kThreads = NT;
    __shared__ uint64_t suf[64];
    __shared__ int sq[64];
    __shared__ int gstart[9];
    __shared__ int16_t posrow[64];
    __shared__ uint8_t Ms[8 * 256];
    uint64_t* X = dsm;                                        // [64][kLuTNW]
    uint64_t* Tb = X + 64 * kLuTNW;                             // [2][256][kLuTNW]
    uint64_t* F = Tb + 2 * 256 * kLuTNW;                        // [8][256] finalize corrections
    uint64_t* cbuf = F + 8 * 256;                             // [kTM]
    int64_t* pbuf = reinterpret_cast<int64_t*>(cbuf + kTM);   // [kTM]

    F2_STAMP(st, 30);
    const int kb = static_cast<int>(ldi(&st->leaf_kb));
    if (kb == 0) return;
    const int64_t r0 = ldi(&st->leaf_r);
    const int64_t row_base = r0 + kb + static_cast<int64_t>(ty) * kTM;
    if (row_base >= A.m && ty != 0) return;
    const int64_t nrows64 = A.m - row_base;
    const int nrows = nrows64 <= 0 ? 0 : (nrows64 < kTM ? static_cast<int>(nrows64) : kTM);
    const int64_t tile_w0 = rw0 + static_cast<int64_t>(tx) * kLuTNW;
    const int ntw = tile_w0 >= rw1 ? 0 : static_cast<int>(rw1 - tile_w0 < kLuTNW ? rw1 - tile_w0 : kLuTNW);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // tables prepared by k_leaf_pivot (depend only on the leaf's pivots)
    for (int i = tid; i < 8 * 256; i += kThreads) F[i] = ldw(&st->leaf_F[0][0] + i);
    for (int i = tid; i < 8 * 256 / 4; i += kThreads)
        reinterpret_cast<uint32_t*>(Ms)[i] = __ldcg(reinterpret_cast<const unsigned int*>(&st->leaf_M[0][0]) + i);
    if (tid < 64) {
        suf[tid] = ldw(&st->ufull[tid]);
        sq[tid] = __ldcg(&st->q[tid]);
        posrow[tid] = -1;
    }
    __syncthreads();
    if (tid < kb) posrow[sq[tid]] = static_cast<int16_t>(tid);
    if (tid <= 8) {
        int lo = 0;
        while (lo < kb && sq[lo] < 8 * tid) ++lo;
        gstart[tid] = lo;
    }
    F2_STAMP(st, 31);

    // 1. finalise the leaf word of the tile's rows -> coefficient words
    for (int i = tid; i < nrows; i += kThreads) {
        const int64_t phys = ldi(pmap + row_base + i);
        uint64_t w = ldw(A.w + phys * A.stride + wl);
#pragma unroll
        for (int g = 0; g < 8; ++g) w ^= F[g * 256 + ((w >> (8 * g)) & 0xffu)];
        cbuf[i] = w;
        pbuf[i] = phys;
        if (tx == 0) A.w[phys * A.stride + wl] = w;
    }
    F2_STAMP(st, 32);
    if (ntw == 0) return;

    // pivot rows' slice of the tile
    for (int i = tid; i < kb * kLuTNW; i += kThreads) {
        const int t = i / kLuTNW, k = i % kLuTNW;
        X[i] = k < ntw ? ldw(A.w + ldi(pmap + r0 + t) * A.stride + tile_w0 + k) : 0ull;
    }
    __syncthreads();

    F2_STAMP(st, 33);
    const int rq = lane >> 3, wp = lane & 7;
    uint64_t acc0[kLuRPT], acc1[kLuRPT];
#pragma unroll
    for (int j = 0; j < kLuRPT; ++j) {
        const int i = warp * 4 * kLuRPT + rq + 4 * j;
        acc0[j] = acc1[j] = 0;
        if (i < nrows) {
            const uint64_t* cr = A.w + pbuf[i] * A.stride + tile_w0;
            if (2 * wp < ntw) acc0[j] = ldw(cr + 2 * wp);
            if (2 * wp + 1 < ntw) acc1[j] = ldw(cr + 2 * wp + 1);
        }
    }

    F2_STAMP(st, 34);
    // 2./3. per group of 8 leaf columns: a table T over the group's pivot rows as they
    // are now; the group's pivot rows and every later row add T[M(c)] (c = the row's
    // coefficient byte, masked below its own pivot for the group's rows), which
    // equals adding the combination of the *solved* group rows (see trsm.cu)
    for (int g = 0; g < 8; ++g) {
        const int g0 = gstart[g], g1 = gstart[g + 1];
        if (g0 == g1) continue;
        const int sh = 8 * g;
        const uint8_t* Mg = Ms + g * 256;
        uint64_t* tb = Tb + (g & 1) * 256 * kLuTNW;
        // table: 4 warps, thread = (16-byte column chunk wp, low nibble el), Gray walk
        if (warp < 4) {
            const int el = tid >> 3;  // 0..15
            uint64_t v0[8], v1[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int r = posrow[sh + b];
                v0[b] = r >= 0 ? X[r * kLuTNW + 2 * wp] : 0ull;
                v1[b] = r >= 0 ? X[r * kLuTNW + 2 * wp + 1] : 0ull;
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
                uint64_t* e = tb + (eh * 16 + el) * kLuTNW + 2 * wp;
                e[0] = l0;
                e[1] = l1;
            }
        }
        __syncthreads();
        for (int i = tid; i < (kb - g0) * kLuTNW; i += kThreads) {
            const int t = g0 + i / kLuTNW, k = i % kLuTNW;
            uint32_t cb = static_cast<uint32_t>(suf[t] >> sh) & 0xffu;
            if (t < g1) cb &= (1u << (sq[t] - sh)) - 1u;
            X[t * kLuTNW + k] ^= tb[Mg[cb] * kLuTNW + k];
        }
#pragma unroll
        for (int j = 0; j < kLuRPT; ++j) {
            const int i = warp * 4 * kLuRPT + rq + 4 * j;
            const unsigned idx = Mg[static_cast<unsigned>(cbuf[i] >> sh) & 0xffu];
            const uint4 v = lu::lds128(tb + idx * kLuTNW + 2 * wp);
            acc0[j] ^= static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32);
            acc1[j] ^= static_cast<uint64_t>(v.z) | (static_cast<uint64_t>(v.w) << 32);
        }
        __syncthreads();
        F2_STAMP(st, 35 + g);
    }

#pragma unroll
    for (int j = 0; j < kLuRPT; ++j) {
        const int i = warp * 4 * kLuRPT + rq + 4 * j;
        if (i < nrows) {
            uint64_t* cr = A.w + pbuf[i] * A.stride + tile_w0;
            if (2 * wp < ntw) cr[2 * wp] = acc0[j];
            if (2 * wp + 1 < ntw) cr[2 * wp + 1] = acc1[j];
        }
    }
    if (ty == 0)
        for (int i = tid; i < kb * kLuTNW; i += kThreads) {
            const int t = i / kLuTNW, k = i % kLuTNW;
            if (k < ntw) A.w[ldi(pmap + r0 + t) * A.stride + tile_w0 + k] = X[i];
        }
}

}  // namespace f2g
