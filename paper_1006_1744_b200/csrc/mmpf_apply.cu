// MMPF table-apply: C ^= A * B for K <= 64 coefficient bits (one word per row), the
// trailing-matrix update of MMPF (add_rows_from_table, proj/src/m4ri.cpp:28-38, with the
// tables of make_table1, proj/src/mmpf.cpp:54-77) and of small addmul products.
//
// HBM-bound streaming: every C row segment is read once and written once, so the kernel
// is shaped for bandwidth, not for table reuse.  The column range is cut into tiles of
// 4096 / ceil2(K / 8) bits (128 KB of tables in SMEM whatever K);
// for a tile a CTA builds ceil(K/8) subset-sum tables of 256 entries in SMEM (entry v of
// table t = XOR of the B rows 8t + b for the set bits b of v, brow < 0 = zero row), then
// streams rows: 16 bytes of C and the row's coefficient word per lane, one 16-byte table
// lookup per coefficient byte, LOP3 XORs, one 16-byte store; 4 row groups in flight per warp.
//
// Work items are (column tile, block of 2048 rows), column-tile major; the persistent
// grid gives every CTA one contiguous run of items, so a CTA rebuilds its tables only
// when its run crosses a column tile.  Rows and the row start come from the device
// (TableApply row modes), so the launch needs no host sync.
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

constexpr int kMThreads = 1024;           // one CTA per SM (128 KB of tables)
constexpr int kMRowBlock = 2048;          // rows per work item
constexpr int kMGroups = 4;               // row groups in flight per warp

__device__ __forceinline__ uint4 xor4m(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }

}  // namespace

// TW: words per column tile; NB: coefficient bits per table (2^NB entries).  The tables take
// 128 KB: with 8-bit tables TW = 64 / ntab (ntab rounded up to a power of two), so K <= 8
// streams 512-byte row segments (4 lines, one DRAM page) and K <= 32 128-byte ones.  For
// 32 < K <= 44 up to 11 4-bit tables at TW = 64 (512-byte segments again) beat 8-bit
// tables at 64-byte segments (K = 33: 2.77 vs 2.32 TB/s over a 1 GiB C); from K = 48 on
// the 4-bit lookups (up to 16 per row) cost more than the short segments (K = 64: 1.85 vs
// 2.05 TB/s), so K > 44 keeps 8-bit tables at TW = 8.  Tiles are aligned to
// absolute multiples of TW words, so every full 16-byte access is aligned; words of a tile
// outside [cw0, cw1) are neither read nor written.
template <int TW, int NB>
__global__ void __launch_bounds__(kMThreads) k_mmpf_apply(TableApply p, int ntab, int rowmajor) {
    constexpr int LPR = TW / 2;               // lanes per row (16 bytes each)
    constexpr int RPI = 32 / LPR;             // rows per warp instruction
    constexpr int U = kMGroups;               // row groups in flight
    constexpr int E = 1 << NB;                // entries per table
    constexpr int NT = 16384 / (E * TW);      // tables that fit 128 KB
    constexpr int KB = NB * NT;               // B rows the tables cover
    using coef_t = typename std::conditional<KB <= 32, uint32_t, uint64_t>::type;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* Bs = reinterpret_cast<uint64_t*>(smem);             // [KB][TW] B rows of the tile
    uint4* T = reinterpret_cast<uint4*>(smem + KB * TW * 8);      // [ntab][E][LPR] uint4

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
    const int64_t nrb = (rows + kMRowBlock - 1) / kMRowBlock;
    const int64_t items = nct * nrb;
    // column-tile major: a contiguous run per CTA (tables rebuilt only where a run crosses a
    // tile); row-block major (rowmajor): item b, b + grid, ... so all CTAs stream nearby rows
    const int64_t i0 = rowmajor ? blockIdx.x : items * blockIdx.x / gridDim.x;
    const int64_t i1 = rowmajor ? items : items * (blockIdx.x + 1) / gridDim.x;
    const int64_t istep = rowmajor ? gridDim.x : 1;
    const uint64_t kmask = p.kbits >= 64 ? ~0ull : (1ull << p.kbits) - 1ull;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane % LPR;     // 16-byte piece of the row segment
    const int rsub = lane / LPR;    // row within a group of RPI
    int64_t cur_ct = -1;
    for (int64_t it = i0; it < i1; it += istep) {
        const int64_t ct = rowmajor ? it % nct : it / nrb, rb = rowmajor ? it / nct : it - ct * nrb;
        const int64_t w0 = wbase + ct * TW;  // first (absolute) C word of the tile
        if (ct != cur_ct) {  // ---- tables for this column tile ----
            __syncthreads();  // previous tile's lookups done
            // the tile's B rows (zero for brow < 0, j >= K or words outside [cw0, cw1)) into Bs
            for (int e = tid; e < KB * TW; e += kMThreads) {
                const int j = e / TW, w = e % TW;
                uint64_t v = 0;
                if (j < p.kbits && w0 + w >= p.cw0 && w0 + w < p.cw1) {
                    const int64_t br = p.brow ? p.brow[j] : p.b_r0 + j;
                    if (br >= 0) v = p.B.w[br * p.B.stride + p.bw0 + (w0 + w - p.cw0)];
                }
                Bs[e] = v;
            }
            // subset sums by doubling: entries [2^b, 2^(b+1)) of table t = entries [0, 2^b) ^ B row NB*t + b
            for (int e = tid; e < ntab * LPR; e += kMThreads) T[(e / LPR) * E * LPR + e % LPR] = make_uint4(0, 0, 0, 0);
            for (int b = 0; b < NB; ++b) {
                __syncthreads();
                const int half = 1 << b, n = ntab * half * LPR;
                for (int e = tid; e < n; e += kMThreads) {
                    const int q = e % LPR, v = (e / LPR) % half, t = e / (half * LPR);
                    const uint4 brow4 = reinterpret_cast<const uint4*>(Bs)[(NB * t + b) * LPR + q];
                    T[(t * E + half + v) * LPR + q] = xor4m(T[(t * E + v) * LPR + q], brow4);
                }
            }
            cur_ct = ct;
            __syncthreads();
        }
        // ---- stream the rows of this block ----
        const int64_t wl = w0 + 2 * sub;  // this lane's first word
        const bool vlo = wl >= p.cw0 && wl < p.cw1, vhi = wl + 1 >= p.cw0 && wl + 1 < p.cw1;
        if (!vlo && !vhi) continue;  // (uniform per lane for the whole item; no barrier below)
        const int64_t rlo = rb * kMRowBlock, rhi = rlo + kMRowBlock < rows ? rlo + kMRowBlock : rows;
        for (int64_t r = rlo + warp * RPI * U; r < rhi; r += static_cast<int64_t>(kMThreads / 32) * RPI * U) {
            uint4 c[U];
            coef_t a[U];
            const int64_t row0 = r + rsub;
            uint64_t* cp0 = p.C.w + (c_r0 + row0) * p.C.stride + wl;
            const uint64_t* ap0 = p.A.w + (a_r0 + row0) * p.A.stride + p.aw0;
            const int64_t cstep = RPI * p.C.stride, astep = RPI * p.A.stride;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                a[u] = 0;
                c[u] = make_uint4(0, 0, 0, 0);
                if (row0 + u * RPI < rhi) {
                    const uint64_t* cp = cp0 + u * cstep;
                    a[u] = static_cast<coef_t>(__ldg(reinterpret_cast<const unsigned long long*>(ap0 + u * astep)) & kmask);
                    if (vlo && vhi) {
                        c[u] = *reinterpret_cast<const uint4*>(cp);
                    } else {
                        const uint64_t v = vlo ? cp[0] : cp[1];
                        c[u] = vlo ? make_uint4(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32), 0, 0)
                                   : make_uint4(0, 0, static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (row0 + u * RPI >= rhi) continue;
                coef_t x = a[u];
                for (int t = 0; t < ntab && x; ++t, x >>= NB)
                    if (x & (E - 1)) c[u] = xor4m(c[u], T[(t * E + static_cast<int>(x & (E - 1))) * LPR + sub]);
                uint64_t* cp = cp0 + u * cstep;
                if (vlo && vhi) {
                    *reinterpret_cast<uint4*>(cp) = c[u];
                } else if (vlo) {
                    cp[0] = static_cast<uint64_t>(c[u].x) | (static_cast<uint64_t>(c[u].y) << 32);
                } else {
                    cp[1] = static_cast<uint64_t>(c[u].z) | (static_cast<uint64_t>(c[u].w) << 32);
                }
            }
        }
    }
}

namespace {
// F2_MMPF_ROWMAJOR=0/1 forces the work order; by default row-block major for one 8-bit
// table (K <= 8: 4.55 vs 4.37 TB/s over a 1 GiB C, the table rebuild per item is cheap),
// column-tile major otherwise (K = 64: 2.04 vs 2.01 TB/s)
int g_mmpf_rowmajor = -1;
bool g_mmpf_nb8 = false;  // F2_MMPF_NB8=1: 32 < K <= 44 with 8-bit tables too (comparison)
template <int TW, int NB>
constexpr size_t mmpf_smem() {
    constexpr int E = 1 << NB, NT = 16384 / (E * TW);
    return static_cast<size_t>(NB * NT) * TW * 8 + static_cast<size_t>(NT) * E * TW * 8;
}
template <int TW, int NB>
void launch_tw(cudaStream_t s, const TableApply& t, int nsm, int ntab) {
    const int rowmajor = g_mmpf_rowmajor >= 0 ? g_mmpf_rowmajor : (NB == 8 && ntab <= 1 ? 1 : 0);
    k_mmpf_apply<TW, NB><<<nsm, kMThreads, mmpf_smem<TW, NB>(), s>>>(t, ntab, rowmajor);
}
template <int TW, int NB>
void setup_tw() {
    cudaFuncSetAttribute(k_mmpf_apply<TW, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(mmpf_smem<TW, NB>()));
}
}  // namespace

void launch_mmpf_apply(cudaStream_t s, const TableApply& t, int nsm) {
    const int ntab = static_cast<int>((t.kbits + 7) / 8);
    if (ntab <= 1) launch_tw<64, 8>(s, t, nsm, ntab);
    else if (ntab <= 2) launch_tw<32, 8>(s, t, nsm, ntab);
    else if (ntab <= 4) launch_tw<16, 8>(s, t, nsm, ntab);
    else if (t.kbits <= 44 && !g_mmpf_nb8) launch_tw<64, 4>(s, t, nsm, static_cast<int>((t.kbits + 3) / 4));
    else launch_tw<8, 8>(s, t, nsm, ntab);
}

void setup_mmpf_apply_kernels() {
    setup_tw<64, 8>();
    setup_tw<32, 8>();
    setup_tw<16, 8>();
    setup_tw<8, 8>();
    setup_tw<64, 4>();
    if (const char* e = std::getenv("F2_MMPF_NB8")) g_mmpf_nb8 = std::atoi(e) != 0;
    if (const char* e = std::getenv("F2_MMPF_ROWMAJOR")) g_mmpf_rowmajor = std::atoi(e);
}

}  // namespace f2g
