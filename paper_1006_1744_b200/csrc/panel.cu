// All leaves of one panel in a single persistent kernel (k_panel_leaves).
//
// The leaf chain of a panel is latency-bound: per 64-column leaf, a one-CTA pivot
// search, then an update of the panel's remaining columns over every row below.  As
// separate launches the fixed launch/drain cost and the serial per-group steps of
// each kernel dominated.  Here one CTA per SM stays resident for the whole panel:
//
//   for each leaf j:
//     CTA 0   pivot search (leaf_pivot_body), then solves the leaf's pivot rows over
//             the rest of the panel, U = L11^{-1} A12 (trsm_lower_left_unit,
//             mul.cpp:109-131), 8 pivot columns at a time, and writes them back
//     -- grid barrier --
//     all     per 512-row tile below the pivots: finalise the leaf word into the L
//             coefficients (the gauss_pls elimination chain, gauss.cpp:47-49, via
//             8 linear 256-entry correction tables) and add, per 8 coefficient bits,
//             one entry of the 256-entry table of combinations of the solved pivot
//             rows (add_rows_from_table, m4ri.cpp:28-38); four group tables are
//             built at once, so a tile needs two table rounds
//     -- grid barrier --
//
// Both table families are linear in the indexing byte, so every CTA derives them
// from 64 basis words instead of loading 4096 entries.  Every cross-CTA value
// (matrix words, pmap, the state) is read with ld.global.cg, and the barrier is
// release/acquire at gpu scope.  The launch is cooperative (all CTAs co-resident);
// the barrier counter is zeroed by a memset node before it.
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"
#include "leaf_body.cuh"

namespace f2g {

namespace {

constexpr int kPT = 1024;                  // threads per CTA
constexpr int kRows = (kPT / 32) * 4 * 4;  // rows per update tile (512): 4 lane groups x 4 rows per warp
constexpr int kW = 16;                     // words of the panel remainder a tile covers (W <= 1024)
constexpr int kTab = 256 * kW;             // one 8-bit group table (CTA 0's fallback solve), words
// dynamic smem: tab[256][kW] (8-bit table of the fallback solve, or the sixteen 4-bit
// tables T4[16][16][kW] of the update) | X[64][kW] | F[8][256]
constexpr size_t kSmem = sizeof(uint64_t) * (kTab + 64 * kW + 8 * 256);
static_assert(kSmem >= sizeof(uint64_t) * (128 + 256) * 15, "CTA 0's fast path scratch");

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
        unsigned v;
        while (true) {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
            if (v >= target) break;
            __nanosleep(64);
        }
        asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    }
    __syncthreads();
}

constexpr unsigned FULL_MASK = 0xffffffffu;

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// Leaf pivot data every phase needs, in shared memory.
struct LeafInfo {
    uint64_t u[64];   // strict pivot words (bits <= pivot cleared)
    uint64_t uf[64];  // full pivot words (L bits, leading 1, S bits)
    int q[64];        // pivot bit positions
    int pos[64];      // bit position -> pivot index, -1
    int gs[9];        // first pivot index of each 8-bit group
    uint64_t fb[64];  // finalize basis: correction for a word whose byte g reads 1 << b
    uint8_t rb[64];   // per group: rows of the inverse 8x8 L block (M[g][e] = xor of rb[8g+b])
    int kb;
    int64_t r0;
    int64_t pmap_hi;  // positions >= pmap_hi are not re-mapped
    int64_t lo;       // first position a worker updates
};

// Loads the current leaf's pivots (st written by CTA 0 before the barrier) and
// derives the two linear table bases.  Ends with __syncthreads.
__device__ void load_leaf(const PlsState* st, LeafInfo& L) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        L.kb = static_cast<int>(ldi(&st->leaf_kb));
        L.r0 = ldi(&st->leaf_r);
        L.pmap_hi = ldi(&st->pmap_hi);
    }
    if (tid < 64) {
        L.u[tid] = ldw(&st->ustrict[tid]);
        L.uf[tid] = ldw(&st->ufull[tid]);
        L.q[tid] = __ldcg(&st->q[tid]);
        L.pos[tid] = -1;
    }
    __syncthreads();
    const int kb = L.kb;
    if (tid < kb) L.pos[L.q[tid]] = tid;
    if (tid <= 8) {  // first pivot of group tid: lower bound of 8*tid in the sorted q
        int lo = 0, hi = kb;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (L.q[mid] < 8 * tid) lo = mid + 1;
            else hi = mid;
        }
        L.gs[tid] = lo;
    }
    __syncthreads();
    if (tid < 64) {  // finalize basis: the gauss_pls chain of group g on the single bit b
        const int g = tid >> 3, b = tid & 7;
        uint64_t x = 1ull << (8 * g + b), corr = 0;
        for (int l = L.gs[g]; l < L.gs[g + 1]; ++l)
            if ((x >> L.q[l]) & 1ull) {
                x ^= L.u[l];
                corr ^= L.u[l];
            }
        L.fb[tid] = corr;
    } else if (tid < 72) {  // inverse 8x8 L block of group g (see trsm.cu)
        const int g = tid - 64;
        uint32_t Rb[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) Rb[b] = 0;
        for (int l = L.gs[g]; l < L.gs[g + 1]; ++l) {
            const int sb = L.q[l] - 8 * g;
            const uint32_t c = static_cast<uint32_t>(L.uf[l] >> (8 * g)) & ((1u << sb) - 1u);
            uint32_t R = 1u << sb;
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if ((c >> b) & 1u) R ^= Rb[b];
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if (b == sb) Rb[b] = R;
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) L.rb[8 * g + b] = static_cast<uint8_t>(Rb[b]);
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned mgroup(const LeafInfo& L, int g, unsigned e) {
    unsigned m = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
        if ((e >> b) & 1u) m ^= L.rb[8 * g + b];
    return m;
}

// CTA 0 after a general-path leaf: the panel TRSM's bytewise map of L11^{-1}
// (st->lmap[leaf], see trsm.cu), computed from the pivot words.  Scratch: 128 words.
__device__ void leaf_lmap(PlsState* st, const LeafInfo& L, int leaf, uint64_t* scratch) {
    const int tid = threadIdx.x, lane = tid & 31;
    uint64_t* rraw = scratch;
    if (tid < 32) {
        const int kb = L.kb;
        uint64_t R0 = 1ull << lane, R1 = 1ull << (lane + 32);  // rows over pivot indices
        for (int tt = 0; tt < kb; ++tt) {
            const int qt = L.q[tt];
            const uint64_t Rt = __shfl_sync(FULL_MASK, tt < 32 ? R0 : R1, tt & 31);
            if (lane > tt && ((L.uf[lane] >> qt) & 1ull)) R0 ^= Rt;
            if (lane + 32 > tt && lane + 32 < kb && ((L.uf[lane + 32] >> qt) & 1ull)) R1 ^= Rt;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int l = lane + 32 * h;
            uint64_t lv = l < kb ? (h ? R1 : R0) : 0ull, r = 0;
            while (lv) {
                const int tt = __ffsll(static_cast<long long>(lv)) - 1;
                lv &= lv - 1;
                r |= 1ull << L.q[tt];
            }
            rraw[l] = r;
        }
    }
    __syncthreads();
    for (int i = tid; i < 8 * 256; i += kPT) {
        const int g = i >> 8, v = i & 255;
        uint64_t x = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int l = L.pos[8 * g + b];
            if (((v >> b) & 1) && l >= 0) x ^= rraw[l];
        }
        st->lmap[leaf][g][v] = x;
    }
    __syncthreads();
}

// CTA 0, after the pivot search: U = L11^{-1} A12 on the pivot rows' words [rw0, rw1),
// written back in place (the pivot rows sit at positions r0 .. r0+kb via pmap).
__device__ void solve_pivot_rows(const Mat& A, int64_t rw0, int64_t rw1, const int64_t* pmap, const LeafInfo& L,
                                 uint64_t* X, uint64_t* tb, PlsState* st_out) {
    const int kb = L.kb, tid = threadIdx.x;
    const int ntw = rw1 > rw0 ? static_cast<int>(rw1 - rw0) : 0;
    if (kb == 0 || ntw == 0) return;
    for (int i = tid; i < kb * kW; i += kPT) {
        const int t = i / kW, k = i % kW;
        X[i] = k < ntw ? ldw(A.w + ldi(pmap + L.r0 + t) * A.stride + rw0 + k) : 0ull;
    }
    __syncthreads();
    for (int g = 0; g < 8; ++g) {
        const int g0 = L.gs[g], g1 = L.gs[g + 1];
        if (g0 == g1) continue;
        // table over the group's rows as they are now: entry e = xor of the rows of e's
        // bits; thread = (2-step segment of the high-nibble Gray walk, low nibble, word pair)
        {
            const int seg = tid >> 7, el = (tid >> 3) & 15, tw = tid & 7;
            uint64_t v0[8], v1[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int r = L.pos[8 * g + b];
                v0[b] = r >= 0 ? X[r * kW + 2 * tw] : 0ull;
                v1[b] = r >= 0 ? X[r * kW + 2 * tw + 1] : 0ull;
            }
            uint64_t l0 = 0, l1 = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((el >> b) & 1) {
                    l0 ^= v0[b];
                    l1 ^= v1[b];
                }
            const int kk = 2 * seg, eh0 = kk ^ (kk >> 1), eh1 = (kk + 1) ^ ((kk + 1) >> 1);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((eh0 >> b) & 1) {
                    l0 ^= v0[4 + b];
                    l1 ^= v1[4 + b];
                }
            uint64_t* e = tb + (eh0 * 16 + el) * kW + 2 * tw;
            e[0] = l0;
            e[1] = l1;
            e = tb + (eh1 * 16 + el) * kW + 2 * tw;  // the Gray step kk -> kk+1 flips bit 0
            e[0] = l0 ^ v0[4];
            e[1] = l1 ^ v1[4];
        }
        __syncthreads();
        // later rows (and the group's own rows, masked below their pivot) add T[M(c)]
        for (int i = tid; i < (kb - g0) * kW; i += kPT) {
            const int t = g0 + i / kW, k = i % kW;
            unsigned cb = static_cast<unsigned>(L.uf[t] >> (8 * g)) & 0xffu;
            if (t < g1) cb &= (1u << (L.q[t] - 8 * g)) - 1u;
            X[t * kW + k] ^= tb[mgroup(L, g, cb) * kW + k];
        }
        __syncthreads();
        F2_STAMP(st_out, 40 + g);
    }
    for (int i = tid; i < kb * kW; i += kPT) {
        const int t = i / kW, k = i % kW;
        if (k < ntw) A.w[ldi(pmap + L.r0 + t) * A.stride + rw0 + k] = X[i];
        st_out->uleaf[t][k] = X[i];
    }
}

// Worker preparation for one leaf (every CTA, after the barrier): one round of
// loads of what CTA 0 published -- pivot columns, the finalize basis and the solved
// pivot rows -- then the finalize tables F[g][v] (xor of the basis over v's bits) and
// the sixteen 4-bit tables T4[g][e] = xor of the solved pivot rows at the pivot
// columns of e's bits in nibble g (word 0 of every entry, the leaf column, is 0).
__device__ void worker_prep(const PlsState::Packet* pk, LeafInfo& L, uint64_t* X, uint64_t* F, uint64_t* T4) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        L.kb = static_cast<int>(ldi(&pk->kb));
        L.r0 = ldi(&pk->r0);
        L.pmap_hi = ldi(&pk->pmap_hi);
        L.lo = ldi(&pk->lo);
    }
    if (tid < 64) {
        L.fb[tid] = ldw(&pk->fb[tid]);
        L.q[tid] = __ldcg(&pk->q[tid]);
        L.pos[tid] = -1;
    }
    for (int i = tid; i < 64 * kW; i += kPT) {
        const int t = i >> 4, w = i & 15;
        X[i] = w == 0 ? 0ull : ldw(&pk->u[t][w - 1]);
    }
    __syncthreads();
    if (tid < L.kb) L.pos[L.q[tid]] = tid;
    for (int i = tid; i < 8 * 256; i += kPT) {
        const int g = i >> 8, v = i & 255;
        uint64_t f = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if ((v >> b) & 1) f ^= L.fb[8 * g + b];
        F[i] = f;
    }
    __syncthreads();
    {  // thread = (nibble group g4, entry e, 4-word quarter wq)
        const int g4 = tid >> 6, e = (tid >> 2) & 15, wq = tid & 3;
        uint64_t v[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = L.pos[4 * g4 + b];
            if (((e >> b) & 1) && r >= 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] ^= X[r * kW + 4 * wq + k];
            }
        }
        uint64_t* d = T4 + (g4 * 16 + e) * kW + 4 * wq;
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = v[k];
    }
    __syncthreads();
}

// One 512-row tile below the pivots (positions r0 + kb + ty*kRows ...): every row's
// panel words wl..pw1 in one load (8 lanes x 2 words per row), the leaf word
// finalised into the L coefficients (the gauss_pls chain of gauss.cpp:47-49 through
// the linear tables F), then 16 nibble lookups add the combination of the solved
// pivot rows (add_rows_from_table, m4ri.cpp:28-38), one store.
__device__ void update_tile(const Mat& A, int64_t wl, int64_t pw1, const int64_t* pmap, const LeafInfo& L, int ty,
                            const uint64_t* F, const uint64_t* T4, const PlsState* st) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t row_base = L.lo + static_cast<int64_t>(ty) * kRows;
    const int64_t nr64 = A.m - row_base;
    const int nrows = nr64 <= 0 ? 0 : (nr64 < kRows ? static_cast<int>(nr64) : kRows);
    const int nw = static_cast<int>(pw1 - wl);  // 1..16 words from the leaf word on
    const int rq = lane >> 3, wp = lane & 7;
    const bool h0 = 2 * wp < nw, h1 = 2 * wp + 1 < nw;
    uint64_t w0[4], w1[4];
    int64_t ph[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = warp * 16 + rq + 4 * j;
        const int64_t pos = row_base + i;
        ph[j] = i < nrows ? (pos < L.pmap_hi ? ldi(pmap + pos) : pos) : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint64_t* rp = A.w + ph[j] * A.stride + wl + 2 * wp;
        w0[j] = ph[j] >= 0 && h0 ? ldw(rp) : 0ull;
        w1[j] = ph[j] >= 0 && h1 ? ldw(rp + 1) : 0ull;
    }
    F2_STAMP(st, 50);
    // finalise: lane x < 16 takes row (rq = x & 3, j = x >> 2), whose leaf word sits
    // on lane 8 * rq (wp == 0) in w0[j]; the coefficient words go back to the groups
    uint64_t c[4];
    {
        const int xr = lane & 3, xj = (lane >> 2) & 3;
        uint64_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t t = __shfl_sync(FULL_MASK, w0[j], 8 * xr);
            v = xj == j ? t : v;
        }
        if (lane < 16) {
#pragma unroll
            for (int g = 0; g < 8; ++g) v ^= F[g * 256 + ((v >> (8 * g)) & 0xffu)];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = __shfl_sync(FULL_MASK, v, rq + 4 * j);
    }
    if (wp == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) w0[j] = c[j];
    }
    F2_STAMP(st, 51);
#pragma unroll
    for (int g4 = 0; g4 < 16; ++g4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned e = static_cast<unsigned>(c[j] >> (4 * g4)) & 15u;
            const uint4 v = lds128(T4 + (g4 * 16 + e) * kW + 2 * wp);
            w0[j] ^= static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32);
            w1[j] ^= static_cast<uint64_t>(v.z) | (static_cast<uint64_t>(v.w) << 32);
        }
    }
    F2_STAMP(st, 52);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (ph[j] < 0) continue;
        uint64_t* rp = A.w + ph[j] * A.stride + wl + 2 * wp;
        if (h0) rp[0] = w0[j];
        if (h1) rp[1] = w1[j];
    }
}

// CTA 0 (non-pipelined schedule): the worker packet from the state the leaf left.
__device__ void publish_from_state(const PlsState* st, PlsState::Packet* pk) {
    const int tid = threadIdx.x;
    __syncthreads();
    if (tid == 0) {
        pk->r0 = st->leaf_r;
        pk->kb = st->leaf_kb;
        pk->lo = st->leaf_r + st->leaf_kb;
        pk->pmap_hi = st->pmap_hi;
    }
    if (tid < 64) {
        pk->q[tid] = st->q[tid];
        pk->fb[tid] = st->fbasis[tid];
    }
    for (int i = tid; i < 64 * 16; i += kPT) (&pk->u[0][0])[i] = (&st->uleaf[0][0])[i];
}

}  // namespace

__global__ void __launch_bounds__(kPT, 1)
k_panel_leaves(Mat A, int64_t pw0, int width, int64_t pw1, PlsState* st, int64_t* P, int64_t* Qp,
               int64_t* pmap, int64_t qcol_off, unsigned* bar) {
    extern __shared__ __align__(16) uint64_t dsm[];
    __shared__ LeafInfo L;
    uint64_t* tab = dsm;  // CTA 0's fallback solve table, or T4
    uint64_t* X = tab + kTab;
    uint64_t* F = X + 64 * kW;
    const int nleaves = (width + 63) / 64;
    unsigned target = 0;
    for (int j = 0; j < nleaves; ++j) {
        const int64_t wl = pw0 + j;
        const int lw = width - 64 * j < 64 ? width - 64 * j : 64;
#ifdef F2_PANEL_PROFILE
        if (threadIdx.x == 0 && blockIdx.x == 0) g_prof_on = (pw0 == 0 && j == 1);
        __syncthreads();
#endif
        F2_STAMP(st, 0);
        if (blockIdx.x == 0) {
            const bool solved = leaf_pivot_body(A, wl, lw, j == 0, j, nleaves * 64, st, P, Qp, pmap, qcol_off, pw1, dsm);
            __syncthreads();
            F2_STAMP(st, 1);
            if (!solved) {  // the general search ran: basis, panel-TRSM map and solve here
                load_leaf(st, L);
                if (threadIdx.x < 64) st->fbasis[threadIdx.x] = L.fb[threadIdx.x];
                leaf_lmap(st, L, j, X);
                solve_pivot_rows(A, wl + 1, pw1, pmap, L, X, tab, st);
            }
            F2_STAMP(st, 2);
            publish_from_state(st, &st->pk[0]);
        }
        grid_barrier(bar, target);
        F2_STAMP(st, 3);
        if (__ldcg(reinterpret_cast<const long long*>(&st->pk[0].kb)) != 0) {
            worker_prep(&st->pk[0], L, X, F, tab);
            F2_STAMP(st, 4);
            const int64_t rows = A.m - L.lo;
            const int ntiles = rows > 0 ? static_cast<int>((rows + kRows - 1) / kRows) : 0;
            for (int ty = blockIdx.x; ty < ntiles; ty += gridDim.x) update_tile(A, wl, pw1, pmap, L, ty, F, tab, st);
        }
        F2_STAMP(st, 5);
#ifdef F2_PANEL_PROFILE
        if (threadIdx.x == 0 && blockIdx.x == 0) g_prof_on = 0;
#endif
        grid_barrier(bar, target);
    }
}

void launch_panel_leaves(cudaStream_t s, const Mat& A, int64_t pw0, int width, int64_t pw1, PlsState* st,
                         int64_t* P, int64_t* Qp, int64_t* pmap, int64_t qcol_off, unsigned* bar, int nsm) {
    cudaMemsetAsync(bar, 0, sizeof(unsigned), s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nsm));
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_panel_leaves, A, pw0, width, pw1, st, P, Qp, pmap, qcol_off, bar);
}

void setup_panel_kernels() {
    cudaFuncSetAttribute(k_panel_leaves, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
}

}  // namespace f2g
