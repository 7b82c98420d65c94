// Table-apply / M4RM kernel: C ^= A * B over GF(2).
//
// This one kernel is both
//   * the MMPF table-apply (add_rows_from_table, proj/src/m4ri.cpp:28-38, fed by
//     make_table1, proj/src/mmpf.cpp:54-77) when K is one 64-bit leaf word: every
//     trailing row adds, per 8 coefficient bits, one row of a 256-entry Gray table
//     of pivot-row combinations; and
//   * the Schur-complement multiply of the blocked PLS (addmul_impl,
//     proj/src/mul.cpp:21-68) when K is a whole panel.
// The coefficient bits are read LSB-first (bits_lsb, mul.cpp:61-66): raw bit j of a
// row's coefficient words selects B row map(j).  In the PLS engine the coefficient
// words are the packed L columns themselves (raw pivot columns; a non-pivot column
// is zero in every row the kernel touches and maps to no B row), so no compaction
// pass exists and the L bits are never rewritten.
//
// CTA tile: 512 rows x 1024 bits of C, accumulated in registers over all of K.
// Per 8-bit chunk of K the CTA builds a 256 x 1024-bit table in SMEM (double
// buffered, 32 KB each) from 8 B rows staged by cp.async four chunks ahead, then
// every row does one 16-byte LDS per thread (8 lanes cover one 128-byte table
// row: conflict-free).  SMEM bandwidth bounds it: 512 lookups + 256 table rows per
// chunk and CTA.
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kRPT = 16;                 // rows per thread
constexpr int kThreads = 256;
constexpr int kTM = (kThreads / 32) * 4 * kRPT;  // 512 rows per CTA
constexpr int kTNW = 16;                 // 64-bit words per tile row (1024 bits)
constexpr int kStages = 4;               // B-row ring depth

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int64_t bmap(const TableApply& p, int64_t j) {
    if (j >= p.kbits) return -1;
    return p.brow ? p.brow[j] : p.b_r0 + j;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) k_table_apply(TableApply p) {
    extern __shared__ __align__(16) uint4 sm4[];
    uint4* Tbuf = sm4;                                                   // [2][256][8]
    uint64_t* ring = reinterpret_cast<uint64_t*>(sm4 + 2 * 256 * 8);   // [kStages][8][kTNW]

    int64_t c_r0 = p.c_r0, a_r0 = p.a_r0;
    if (p.row_mode == ROWS_AFTER_LEAF) {
        if (p.st->leaf_kb == 0) return;
        c_r0 = a_r0 = p.st->leaf_r + p.st->leaf_kb;
    } else if (p.row_mode == ROWS_AFTER_PANEL) {
        if (p.st->panel_kb == 0) return;
        c_r0 = a_r0 = p.st->panel_r + p.st->panel_kb;
    }
    const int64_t row_base = c_r0 + static_cast<int64_t>(blockIdx.y) * kTM;
    if (row_base >= p.c_r1) return;
    const int64_t tile_w0 = p.cw0 + static_cast<int64_t>(blockIdx.x) * kTNW;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rg = lane >> 3, wp = lane & 7;
    const int64_t cwa = tile_w0 + 2 * wp, cwb = cwa + 1;
    const bool va = cwa < p.cw1, vb = cwb < p.cw1;

    uint64_t acc0[kRPT], acc1[kRPT];
    uint64_t aw[kRPT], an[kRPT];
    const int64_t nch = (p.kbits + 7) / 8;

#pragma unroll
    for (int i = 0; i < kRPT; ++i) {
        const int64_t row = row_base + warp * 64 + rg + 4 * i;
        const bool rv = row < p.c_r1;
        const uint64_t* cr = p.C.w + row * p.C.stride;
        acc0[i] = (rv && va) ? cr[cwa] : 0ull;
        acc1[i] = (rv && vb) ? cr[cwb] : 0ull;
        an[i] = rv ? p.A.w[(a_r0 + (row - c_r0)) * p.A.stride + p.aw0] : 0ull;
        aw[i] = 0;
    }

    // stage B rows of chunk c into ring slot c % kStages (threads 0..127, one word each)
    auto issue = [&](int64_t c) {
        if (tid < 8 * kTNW) {
            const int b = tid >> 4, k = tid & 15;
            const int64_t br = bmap(p, c * 8 + b);
            const int64_t wcol = tile_w0 + k;
            const bool ok = br >= 0 && wcol < p.cw1;
            const uint64_t* src = ok ? p.B.w + br * p.B.stride + (p.bw0 + (wcol - p.cw0)) : p.B.w;
            cp_async8(ring + ((c % kStages) * 8 + b) * kTNW + k, src, ok);
        }
    };
    auto live = [&](int64_t c) {
        bool any = false;
#pragma unroll
        for (int b = 0; b < 8; ++b) any |= bmap(p, c * 8 + b) >= 0;
        return any;
    };
    // 256-entry table of chunk c into buffer buf: entry e = xor of B rows b with bit b of e
    auto build = [&](int buf, int64_t c) {
        const uint64_t* rs = ring + (c % kStages) * 8 * kTNW;
        const int el = tid >> 3;  // low 5 bits of the entry
        uint64_t v0[8], v1[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            v0[b] = rs[b * kTNW + 2 * wp];
            v1[b] = rs[b * kTNW + 2 * wp + 1];
        }
        uint64_t l0 = 0, l1 = 0;
#pragma unroll
        for (int b = 0; b < 5; ++b)
            if ((el >> b) & 1) {
                l0 ^= v0[b];
                l1 ^= v1[b];
            }
        uint64_t h0 = 0, h1 = 0;
        uint4* tb = Tbuf + buf * 256 * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k) {
                const int b = 5 + ((k & 1) ? 0 : ((k & 2) ? 1 : 2));  // 5 + ctz(k), folded
                h0 ^= v0[b];
                h1 ^= v1[b];
            }
            const int eh = k ^ (k >> 1);
            const uint64_t x0 = l0 ^ h0, x1 = l1 ^ h1;
            tb[(eh * 32 + el) * 8 + wp] = make_uint4(static_cast<unsigned>(x0), static_cast<unsigned>(x0 >> 32),
                                                     static_cast<unsigned>(x1), static_cast<unsigned>(x1 >> 32));
        }
    };

    for (int64_t c = 0; c < 3; ++c) {
        if (c < nch) issue(c);
        cp_async_commit();
    }
    cp_async_wait<2>();
    __syncthreads();
    if (nch > 0 && live(0)) build(0, 0);

    for (int64_t c = 0; c < nch; ++c) {
        if (c + 3 < nch) issue(c + 3);
        cp_async_commit();
        if ((c & 7) == 0) {
            const int64_t g1 = (c >> 3) + 1;
#pragma unroll
            for (int i = 0; i < kRPT; ++i) {
                aw[i] = an[i];
                const int64_t row = row_base + warp * 64 + rg + 4 * i;
                if (g1 < p.kw && row < p.c_r1)
                    an[i] = p.A.w[(a_r0 + (row - c_r0)) * p.A.stride + p.aw0 + g1];
            }
        }
        cp_async_wait<2>();
        __syncthreads();
        if (c + 1 < nch && live(c + 1)) build(static_cast<int>((c + 1) & 1), c + 1);
        if (live(c)) {
            const uint4* tb = Tbuf + (c & 1) * 256 * 8 + wp;
            const int sh = 8 * static_cast<int>(c & 7);
#pragma unroll
            for (int i = 0; i < kRPT; ++i) {
                const unsigned idx = static_cast<unsigned>(aw[i] >> sh) & 0xffu;
                const uint4 v = tb[idx * 8];
                acc0[i] ^= static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32);
                acc1[i] ^= static_cast<uint64_t>(v.z) | (static_cast<uint64_t>(v.w) << 32);
            }
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < kRPT; ++i) {
        const int64_t row = row_base + warp * 64 + rg + 4 * i;
        if (row < p.c_r1) {
            uint64_t* cr = p.C.w + row * p.C.stride;
            if (va) cr[cwa] = acc0[i];
            if (vb) cr[cwb] = acc1[i];
        }
    }
}

static size_t table_apply_smem() { return sizeof(uint4) * 2 * 256 * 8 + sizeof(uint64_t) * kStages * 8 * kTNW; }

void launch_table_apply(cudaStream_t s, const TableApply& t, int nsm) {
    (void)nsm;
    if (t.cw1 <= t.cw0 || t.kbits <= 0) return;
    const int64_t lo = t.row_mode == ROWS_STATIC ? t.c_r0 : 0;
    const int64_t rows = t.c_r1 - lo;
    if (rows <= 0) return;
    dim3 grid(static_cast<unsigned>((t.cw1 - t.cw0 + kTNW - 1) / kTNW), static_cast<unsigned>((rows + kTM - 1) / kTM));
    k_table_apply<<<grid, kThreads, table_apply_smem(), s>>>(t);
}

void setup_m4rm_kernels() {
    cudaFuncSetAttribute(k_table_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(table_apply_smem()));
}

}  // namespace f2g
