// MMPF table-apply: C ^= A * B for K <= 64 coefficient bits (one word per row), the
// trailing-matrix update of MMPF (add_rows_from_table, proj/src/m4ri.cpp:28-38, with the
// tables of make_table1, proj/src/mmpf.cpp:54-77) and of small addmul products.
//
// HBM-bound streaming: every C row segment is read once and written once.  The column
// range is cut into 1024-bit tiles; for a tile a CTA builds subset-sum tables in SMEM
// (entry v of table t = XOR of the B rows NB*t + b for the set bits b of v; brow < 0 or
// j >= K: zero row), then streams 128-byte row segments: 8 lanes per row, 16 bytes of C
// and the row's coefficient word per lane, one 16-byte table lookup per NB coefficient
// bits, LOP3 XORs, one 16-byte store; 8 row groups in flight per warp.  Work items are
// (column tile, block of rows); rows and the row start come from the device (TableApply
// row modes), so the launch needs no host sync.
//
// Measured over a 1 GiB C (65536 x 131072, tools/ta_bench.py, bench.py table_apply_hbm):
// K = 8: 5.49 TB/s, K = 33: 5.28, K = 64: 4.24 (of a measured 6.55 TB/s copy); the
// round-1 layout (512- to 4096-bit tiles, 1024 threads, per-table loop) ran 4.54 / 2.69 /
// 2.04 -- instruction-bound at 334 instructions per 4 rows (ncu: issue slots 65 %).
#include <cstdint>
#include <cstdlib>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {
__device__ __forceinline__ uint4 xor4m(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }
}  // namespace

// K <= 24: ceil(K/8) tables of 256 entries (8 bits, 32 KB each); K > 24: ceil(K/7) tables
// of 128 entries (7 bits, 16 KB each, up to 160 KB).  Entries are 128 bytes: a row segment
// is one 128-byte line read by 8 lanes, and a table lookup by those 8 lanes is one
// conflict-free 128-byte SMEM wavefront.  The tables sit at a shared address aligned to
// one table's size TB, so the address of entry v of table t for a lane is
//   ((coef >> (NB*t - 7)) & ((2^NB - 1) << 7)) | base_lane,  plus the immediate t * TB:
// a lookup costs a shift, a LOP3 and an LDS, and two lookups fold into C with three-input
// LOP3 XORs.  Coefficient bits past K select B rows staged as zero, so no masking.
// Work order: row-block major (item b, b + grid, ...), so all CTAs stream nearby rows.
constexpr int k7Lpr = 8;                 // lanes per row (16 bytes each): 128-byte segments
constexpr int k7Rpi = 32 / k7Lpr;        // rows per warp instruction
constexpr int k7U = 8;                   // row groups in flight per warp
constexpr int k7Threads = 512;           // one CTA per SM (up to 160 KB of tables)
template <int NB>
__host__ __device__ constexpr int k7TableBytes() { return (1 << NB) * 128; }  // one NB-bit table at 1024 bits
template <int NB>
constexpr size_t k7Smem(int ntab) { return static_cast<size_t>(ntab + 1) * k7TableBytes<NB>() + NB * ntab * 128; }

template <int NB, int T>
__device__ __forceinline__ uint32_t k7_off(uint64_t a) {
    constexpr int sh = NB * T;
    return (sh >= 7 ? static_cast<uint32_t>(a >> (sh - 7)) : static_cast<uint32_t>(a) << 7) & (((1u << NB) - 1) << 7);
}

template <int NB, int T>
__device__ __forceinline__ uint4 k7_lds(uint32_t base, uint64_t a) {
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4 + %5];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "r"(k7_off<NB, T>(a) | base), "n"(T * k7TableBytes<NB>()));
    return v;
}

template <int NB, int T, int NTAB>
__device__ __forceinline__ void k7_apply(uint4& c, uint32_t base, uint64_t a) {
    if constexpr (T + 1 < NTAB) {
        const uint4 x = k7_lds<NB, T>(base, a), y = k7_lds<NB, T + 1>(base, a);
        c = make_uint4(c.x ^ x.x ^ y.x, c.y ^ x.y ^ y.y, c.z ^ x.z ^ y.z, c.w ^ x.w ^ y.w);
        k7_apply<NB, T + 2, NTAB>(c, base, a);
    } else if constexpr (T < NTAB) {
        const uint4 x = k7_lds<NB, T>(base, a);
        c = xor4m(c, x);
    }
}

template <int NB, int NTAB>
__global__ void __launch_bounds__(k7Threads, 1) k_mmpf_apply7(TableApply p, int rblock) {
    constexpr int TW = 16, KB = NB * NTAB, E = 1 << NB, TB = k7TableBytes<NB>();
    constexpr int U = k7U;
    extern __shared__ __align__(128) unsigned char smem[];
    // tables at the first TB-aligned shared address (so the entry offset can be OR-ed into
    // the lane's base), the staged B rows after them
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const uint32_t tpad = ((sbase + (TB - 1u)) & ~(TB - 1u)) - sbase;
    uint4* T = reinterpret_cast<uint4*>(smem + tpad);                     // [NTAB][E][8]
    uint64_t* Bs = reinterpret_cast<uint64_t*>(smem + tpad + NTAB * TB);  // [KB][16]

    int64_t c_r0 = p.c_r0, a_r0 = p.a_r0;
    if (p.row_mode == ROWS_AFTER_LEAF) {
        if (p.st->leaf_kb == 0) return;
        c_r0 = a_r0 = p.st->leaf_r + p.st->leaf_kb;
    } else if (p.row_mode == ROWS_AFTER_PANEL) {
        const int64_t pr = p.rk ? p.rk[0] : p.st->panel_r, pk = p.rk ? p.rk[1] : p.st->panel_kb;
        if (pk == 0) return;
        c_r0 = a_r0 = pr + pk;
    }
    const int64_t rows = p.c_r1 - c_r0;
    if (rows <= 0) return;
    const int64_t wbase = p.cw0 / TW * TW;
    const int64_t nct = (p.cw1 - wbase + TW - 1) / TW;
    const int64_t nrb = (rows + rblock - 1) / rblock;
    const int64_t items = nct * nrb;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane % k7Lpr, rsub = lane / k7Lpr;
    const uint32_t lbase = sbase + tpad + 16u * sub;  // this lane's 16 bytes of entry 0, table 0
    const int64_t cs = p.C.stride, as = p.A.stride;
    constexpr int kWarpRows = k7Rpi * U;                       // rows per warp per iteration
    constexpr int kStepRows = (k7Threads / 32) * kWarpRows;    // rows per CTA per iteration
    int64_t cur_ct = -1;
    // row-block major: item b, b + grid, ...: all CTAs stream nearby rows
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t ct = it % nct, rb = it / nct;
        const int64_t w0 = wbase + ct * TW;
        if (ct != cur_ct) {
            __syncthreads();
            for (int e = tid; e < KB * TW; e += k7Threads) {
                const int j = e / TW, w = e % TW;
                uint64_t v = 0;
                if (j < p.kbits && w0 + w >= p.cw0 && w0 + w < p.cw1) {
                    const int64_t br = p.brow ? p.brow[j] : p.b_r0 + j;
                    if (br >= 0) v = p.B.w[br * p.B.stride + p.bw0 + (w0 + w - p.cw0)];
                }
                Bs[e] = v;
            }
            for (int e = tid; e < NTAB * k7Lpr; e += k7Threads) T[(e / k7Lpr) * E * k7Lpr + e % k7Lpr] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
            for (int b = 0; b < NB; ++b) {
                __syncthreads();
                const int half = 1 << b, n = NTAB * half * k7Lpr;
                for (int e = tid; e < n; e += k7Threads) {
                    const int q = e % k7Lpr, v = (e / k7Lpr) % half, t = e / (half * k7Lpr);
                    const uint4 brow4 = reinterpret_cast<const uint4*>(Bs)[(NB * t + b) * k7Lpr + q];
                    T[(t * E + half + v) * k7Lpr + q] = xor4m(T[(t * E + v) * k7Lpr + q], brow4);
                }
            }
            cur_ct = ct;
            __syncthreads();
        }
        const int64_t wl = w0 + 2 * sub;
        const bool vlo = wl >= p.cw0 && wl < p.cw1, vhi = wl + 1 >= p.cw0 && wl + 1 < p.cw1;
        if (!vlo && !vhi) continue;
        const int64_t rlo = rb * rblock, rhi = rlo + rblock < rows ? rlo + rblock : rows;
        int64_t r = rlo + warp * kWarpRows + rsub;  // this lane's row of group 0
        uint64_t* cp = p.C.w + (c_r0 + r) * cs + wl;
        const uint64_t* ap = p.A.w + (a_r0 + r) * as + p.aw0;
        const int64_t cu = k7Rpi * cs, au = k7Rpi * as;
        if (vlo && vhi) {
            // full 16-byte pieces: every group of the iteration in range, loads first
            for (; r + (U - 1) * k7Rpi < rhi; r += kStepRows, cp += kStepRows * cs, ap += kStepRows * as) {
                uint4 c[U];
                uint64_t a[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    a[u] = __ldg(reinterpret_cast<const unsigned long long*>(ap + u * au));
                    c[u] = __ldcs(reinterpret_cast<const uint4*>(cp + u * cu));
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    k7_apply<NB, 0, NTAB>(c[u], lbase, a[u]);
                    __stcs(reinterpret_cast<uint4*>(cp + u * cu), c[u]);
                }
            }
            for (int u = 0; u < U; ++u) {  // the block's last partial iteration
                if (r + u * k7Rpi >= rhi) break;
                uint4 c = __ldcs(reinterpret_cast<const uint4*>(cp + u * cu));
                k7_apply<NB, 0, NTAB>(c, lbase, __ldg(reinterpret_cast<const unsigned long long*>(ap + u * au)));
                __stcs(reinterpret_cast<uint4*>(cp + u * cu), c);
            }
        } else {
            // one word of the piece inside [cw0, cw1) (tile edges)
            const int h = vlo ? 0 : 1;
            for (; r < rhi; r += kStepRows, cp += kStepRows * cs, ap += kStepRows * as) {
                for (int u = 0; u < U && r + u * k7Rpi < rhi; ++u) {
                    uint64_t* q = cp + u * cu;
                    const uint64_t v = q[h];
                    uint4 c = h == 0 ? make_uint4(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32), 0, 0)
                                     : make_uint4(0, 0, static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
                    k7_apply<NB, 0, NTAB>(c, lbase, __ldg(reinterpret_cast<const unsigned long long*>(ap + u * au)));
                    q[h] = h == 0 ? static_cast<uint64_t>(c.x) | (static_cast<uint64_t>(c.y) << 32)
                                  : static_cast<uint64_t>(c.z) | (static_cast<uint64_t>(c.w) << 32);
                }
            }
        }
    }
}

namespace {

template <int NB, int NTAB>
void launch_k7n(cudaStream_t s, const TableApply& t, int nsm) {
    // rows per item: 2048 while the table rebuild is cheap (K <= 16: 5.5 vs 5.3 TB/s at
    // 8192), 8192 above (K = 64: 4.25 vs 3.60 TB/s at 2048), over a 1 GiB C
    const int rb = NB * NTAB <= 16 ? 2048 : 8192;  // rows per work item
    k_mmpf_apply7<NB, NTAB><<<nsm, k7Threads, k7Smem<NB>(NTAB), s>>>(t, rb);
}
template <int NB, int NTAB>
void setup_k7() {
    cudaFuncSetAttribute(k_mmpf_apply7<NB, NTAB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(k7Smem<NB>(NTAB)));
}
}  // namespace

// 8-bit tables for K <= 24 (1-3 tables, 32-96 KB), 7-bit tables above (4-10, 64-160 KB):
// K = 32 on four 8-bit tables ran at 4.43 TB/s, K = 33 on five 7-bit ones at 5.28
void launch_mmpf_apply(cudaStream_t s, const TableApply& t, int nsm) {
    const int k = static_cast<int>(t.kbits);
    if (k <= 24) {
        switch ((k + 7) / 8) {
            case 1: launch_k7n<8, 1>(s, t, nsm); break;
            case 2: launch_k7n<8, 2>(s, t, nsm); break;
            default: launch_k7n<8, 3>(s, t, nsm); break;
        }
        return;
    }
    switch ((k + 6) / 7) {
        case 4: launch_k7n<7, 4>(s, t, nsm); break;
        case 5: launch_k7n<7, 5>(s, t, nsm); break;
        case 6: launch_k7n<7, 6>(s, t, nsm); break;
        case 7: launch_k7n<7, 7>(s, t, nsm); break;
        case 8: launch_k7n<7, 8>(s, t, nsm); break;
        case 9: launch_k7n<7, 9>(s, t, nsm); break;
        default: launch_k7n<7, 10>(s, t, nsm); break;
    }
}

void setup_mmpf_apply_kernels() {
    setup_k7<8, 1>();
    setup_k7<8, 2>();
    setup_k7<8, 3>();
    setup_k7<7, 4>();
    setup_k7<7, 5>();
    setup_k7<7, 6>();
    setup_k7<7, 7>();
    setup_k7<7, 8>();
    setup_k7<7, 9>();
    setup_k7<7, 10>();
}

}  // namespace f2g
