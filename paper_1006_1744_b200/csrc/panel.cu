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

// CTA 0 waits for the other CTAs' arrivals at the barrier after `target` (the next one).
__device__ __forceinline__ void await_workers(const unsigned* bar, unsigned target) {
    unsigned v;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target + gridDim.x - 1);
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (blockIdx.x == 0) {
        // CTA 0 (the critical path, nearly always the last to arrive) waits for the others'
        // arrivals only, then arrives without waiting for its own to land: no CTA's next
        // round can begin before it, so target - 1 arrivals are this round's
        if (threadIdx.x == 0) {
            await_workers(bar, target - gridDim.x);
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
        }
        __syncthreads();
        return;
    }
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
    // lanes whose words lie right of the panel read their row's first entry instead: the
    // same address as lane wp = 0, so the lookup costs no extra shared-memory wavefront
    const int wpa = h0 ? wp : 0;
#pragma unroll
    for (int g4 = 0; g4 < 16; ++g4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned e = static_cast<unsigned>(c[j] >> (4 * g4)) & 15u;
            const uint4 v = lds128(T4 + (g4 * 16 + e) * kW + 2 * wpa);
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



// ---- pipelined schedule (k_panel_pipe) --------------------------------------------------
//
// CTA 0 keeps the 128-row window of the current order in shared memory (row form,
// the panel's 16 words per row) and carries it from leaf to leaf: after leaf j the
// rows that did not become pivots stay, the leaf's pivots are replaced by the next
// kb rows of the order, and CTA 0 itself applies leaf j's update to all 128.  So the
// search for leaf j+1 needs nothing from the other CTAs, which meanwhile apply leaf
// j to every row past the next window.  One grid barrier per leaf, and the row
// updates run concurrently with the next pivot search.  A leaf the window search
// cannot decide inside the window (rank-deficient / sparse inputs) falls back to the
// general search on the global matrix: CTA 0 writes its window back, waits for the
// workers, searches, then the workers update everything before a fresh window.
namespace {

constexpr int kPW = 128;  // window slots
struct PipeSmem {
    uint64_t win[2][kPW][16];  // window rows, panel words pw0 .. pw0+15 (double buffered)
    uint64_t T[16 * 16 * kW];  // 4-bit tables over the last fast leaf's solved rows
    uint64_t F[8 * 256];       // its finalize tables
    uint64_t t16[256 * 15];    // solve scratch: 4-bit tables over the pivot rows' rest words
    uint64_t U[64 * 16];       // this leaf's solved rows (word 0 = 0, 1.. = rest words)
};
constexpr size_t kPipeSmem = sizeof(PipeSmem) > kSmem ? sizeof(PipeSmem) : kSmem;

enum PipeState : int64_t { S_FRESH = 0, S_CARRY = 1, S_GENERAL = 2, S_IDLE = 3, S_FINAL = 4, S_DONE = 5 };

struct PipeStatic {  // CTA 0's persistent window bookkeeping
    int64_t wphys[2][kPW];
    int srcprev[kPW];
    int cs[kPW];
};

// Leaf `leafp`'s update of words [k0, k1) of every window slot: the combination of its
// solved rows selected by the slot's coefficient word (S.t16 scratch), through the tables T.
// Threads tid, tid + nth, ... of one (slot, word) item each.
__device__ __forceinline__ void pipe_phase2(PipeSmem& S, int pb, int leafp, int k0, int k1, int tid, int nth) {
    const int nk = k1 - k0;
    if (nk <= 0) return;
    for (int i = tid; i < kPW * nk; i += nth) {
        const int sl = i / nk, k = k0 + (i - sl * nk);
        const uint64_t c = S.t16[sl];
        uint64_t v = S.win[pb][sl][k];
#pragma unroll
        for (int g4 = 0; g4 < 16; ++g4) v ^= S.T[(g4 * 16 + ((c >> (4 * g4)) & 15u)) * kW + (k - leafp)];
        S.win[pb][sl][k] = v;
    }
}

// Window for leaf `leaf` into buffer `pb`: fresh from the global matrix (every leaf
// before it applied there), or carried from buffer pb^1 (leaf-1's window, kbp pivots,
// srcprev) plus new rows, with leaf-1's update applied by CTA 0.
__device__ void pipe_build_window(const Mat& A, int64_t pw0, int nwp, const int64_t* pmap, PlsState* st,
                                  PipeSmem& S, PipeStatic& Z, int pb, bool carry, int kbp, int leafp,
                                  int64_t pmap_hi, bool all_words) {
    const int tid = threadIdx.x;
    const int64_t base = st->r;  // position of slot 0
    const int64_t m = A.m;
    // phase 0: sources (previous window slot or a global row) and physical rows
    for (int i = tid; i < kPW * 16; i += kPT) {
        const int sl = i >> 4, k = i & 15;
        int64_t ph;
        uint64_t v = 0;
        if (carry && sl < kPW - kbp) {
            const int ss = Z.srcprev[kbp + sl];
            ph = Z.wphys[pb ^ 1][ss];
            v = S.win[pb ^ 1][ss][k];
        } else {
            const int64_t pos = base + sl;
            ph = pos < m ? (pos < pmap_hi ? ldi(pmap + pos) : pos) : -1;
            v = (ph >= 0 && k < nwp) ? ldw(A.w + ph * A.stride + pw0 + k) : 0ull;
        }
        S.win[pb][sl][k] = v;
        if (k == 0) Z.wphys[pb][sl] = ph;
    }
    if (!carry) {
        __syncthreads();
        return;
    }
    __syncthreads();
    // phase 1: leaf-1's word of every slot -> its L coefficients (finalize chain)
    if (tid < kPW) {
        uint64_t x = S.win[pb][tid][leafp];
#pragma unroll
        for (int g = 0; g < 8; ++g) x ^= S.F[g * 256 + ((x >> (8 * g)) & 0xffu)];
        S.win[pb][tid][leafp] = x;
        Z.cs[tid] = 0;
        reinterpret_cast<uint64_t*>(S.t16)[tid] = x;  // coefficient words (scratch)
    }
    __syncthreads();
    // phase 2: the words right of leaf-1 add the combination of its solved rows -- here only
    // the next leaf's word, which its search reads; pipe_fast_leaf's idle warps update the
    // others beside the search (pipe_phase2), unless all_words (the final write-back)
    if (all_words) {
        pipe_phase2(S, pb, leafp, leafp + 1, nwp, tid, kPT);
    } else if (tid < kPW && leafp + 1 < nwp) {
        pipe_phase2(S, pb, leafp, leafp + 1, leafp + 2, tid, kPT);
    }
    __syncthreads();
}

// A worker CTA: the panel TRSM's bytewise L11^{-1} map of the packet's leaf (trsm.cu),
// lmap[g][v] = xor over bits b of v of the L11^{-1} row of the pivot at column 8g+b.
__device__ void pipe_worker_lmap(PlsState* st, const PlsState::Packet* pk, uint64_t* scratch) {
    const int tid = threadIdx.x;
    uint64_t* rraw = scratch;                                  // [64]
    int* posc = reinterpret_cast<int*>(scratch + 64);          // [64]
    int* q = posc + 64;                                        // [64]
    const int kb = static_cast<int>(ldi(&pk->kb));
    const int leaf = static_cast<int>(ldi(&pk->leaf));
    if (tid < 64) {
        q[tid] = __ldcg(&pk->q[tid]);
        posc[tid] = -1;
    }
    __syncthreads();
    if (tid < 64) {
        uint64_t lv = tid < kb ? ldw(&pk->linv[tid]) : 0ull, r = 0;
        while (lv) {
            const int tt = __ffsll(static_cast<long long>(lv)) - 1;
            lv &= lv - 1;
            r |= 1ull << q[tt];
        }
        rraw[tid] = r;
        if (tid < kb) posc[q[tid]] = tid;
    }
    __syncthreads();
    for (int i = tid; i < 8 * 256; i += kPT) {
        const int g = i >> 8, v = i & 255;
        uint64_t x = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int l = posc[8 * g + b];
            if (((v >> b) & 1) && l >= 0) x ^= rraw[l];
        }
        st->lmap[leaf][g][v] = x;
    }
    __syncthreads();
}

__device__ void pipe_write_back(const Mat& A, int64_t pw0, int nwp, const PipeSmem& S, const PipeStatic& Z, int pb) {
    for (int i = threadIdx.x; i < kPW * 16; i += kPT) {
        const int sl = i >> 4, k = i & 15;
        const int64_t ph = Z.wphys[pb][sl];
        if (ph >= 0 && k < nwp) A.w[ph * A.stride + pw0 + k] = S.win[pb][sl][k];
    }
}

// Row-form search (leaf_body.cuh, row_pivots) of leaf `leaf` on window buffer pb; on success publishes every
// output (P, Q, pmap moves, pivot rows' slices, state, panel-TRSM map, worker packet)
// and the carry tables, and returns kb; -1 when the window cannot decide a column.
__device__ int pipe_fast_leaf(const Mat& A, int64_t pw0, int nwp, int leaf, int lw, PlsState* st, int64_t* P,
                              int64_t* Qp, int64_t* pmap, int64_t qcol_off, PipeSmem& S, PipeStatic& Z, int pb,
                              PlsState::Packet* pk, int nleaves, bool carried, bool past_zero, bool& search4) {
    __shared__ FastSmem F;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m = A.m, stride = A.stride;
    const int64_t base = st->r;
    const int64_t span = m - base;
    const int nrest = nwp - leaf - 1;  // rest words right of the leaf
    const bool first = leaf == 0;
    const int64_t wl = pw0 + leaf;
    F2_STAMP(st, 16);
    F2_CLK(const bool clk = pw0 == 0 && leaf == 2 && tid == 0; long long c0 = clock64();)
    if (warp == 0) {
        // the first 96 slots decide a dense leaf; all 128 when they cannot (rank-deficient / sparse)
        // (search4, sticky for the panel: a leaf needed all 128, so will the next ones)
        if (lane == 0) F.used4 = 0;
        if (search4 || row_pivots<3>(F, &S.win[pb][0][leaf], lw, base + 96 < m) < 0) {
            __syncwarp();
            row_pivots<4>(F, &S.win[pb][0][leaf], lw, base + kPW < m && !past_zero);
            if (lane == 0) F.used4 = 1;
        }
    }
    // meanwhile the other warps finish the carried window: the previous leaf's update of
    // the words right of this leaf's (pipe_build_window did this leaf's word)
    // (warps 3, 7, ..., 31 only: the fourth scheduler, away from the searching warp 0)
    if ((warp & 3) == 3 && carried) pipe_phase2(S, pb, leaf - 1, leaf + 1, nwp, (warp >> 2) * 32 + (tid & 31), kPT / 4);
    __syncthreads();
    F2_CLK(if (clk) { st->dbg[20] = clock64() - c0; st->dbg[29] = F.clk[1] - F.clk[0]; })
    F2_STAMP(st, 18);
    const int kb = F.final_kb;
    if (F.used4) search4 = true;
    if (kb < 0) return -1;

    // warps 0-1: L11^-1, while the others derive everything that does not need it (the slot
    // sources and the column -> pivot map came with the search)
    if (warp < 2) {
        pair_linv_rows(F, kb);
        F2_CLK(if (pw0 == 0 && leaf == 2 && tid == 0) st->dbg[28] = clock64() - c0;)
    } else if (tid < 128) {
        // finalize basis: what the unit word e (bit e of the leaf word) receives from the pivots
        // of its own byte group, applied in column order (x has bit q: x ^= U above q)
        const int e = tid - 64, g = e >> 3;
        uint64_t uw[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int l = F.posc[8 * g + b];
            uw[b] = l >= 0 ? F.uf[l] & above(8 * g + b) : 0ull;
        }
        uint64_t x = 1ull << e, corr = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if ((x >> (8 * g + b)) & 1ull) {
                x ^= uw[b];
                corr ^= uw[b];
            }
        pk->fb[e] = corr;
        F.fbas[e] = corr;
        F2_CLK(if (pw0 == 0 && leaf == 2 && e == 63) st->dbg[30] = clock64() - c0;)
    } else if (tid >= 256 && tid < 320) {
        const int l = tid - 256;
        const bool in = l < kb;
        const int q = in ? F.step_c[l] : 64;
        st->ustrict[l] = in ? F.uf[l] & above(q) : 0ull;
        st->ufull[l] = in ? F.uf[l] : 0ull;
        st->q[l] = q;
        pk->q[l] = q;
    } else if (tid >= 320 && tid < 576) {
        // 4-bit tables over A12 (the pivot rows' pre-leaf rest words, pivot order): they need
        // only the slot sources, so they are built here, beside L11^-1.  Thread = (group g of
        // four pivots, rest word k): four loads, then the sixteen subset sums in Gray order
        const int g = (tid - 320) >> 4, k = (tid - 320) & 15;
        if (k < nrest) {
            uint64_t v[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) v[b] = 4 * g + b < kb ? S.win[pb][F.src[4 * g + b]][leaf + 1 + k] : 0ull;
            uint64_t x = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (i) x ^= v[(i & 1) ? 0 : ((i & 2) ? 1 : ((i & 4) ? 2 : 3))];  // the bit that flips in i ^ (i >> 1)
                S.t16[((g << 4) | (i ^ (i >> 1))) * 15 + k] = x;
            }
        }
    }
    if (first)
        for (int i = tid; i < nleaves * 64; i += kPT) st->brow[i] = -1;
    __syncthreads();
    F2_CLK(if (clk) st->dbg[25] = clock64() - c0;)
    F2_STAMP(st, 19);
    // solved rest words U_l = sum over t of Linv[l][t] A12_t
    for (int i = tid; i < 64 * 16; i += kPT) {
        const int l = i >> 4, k = i & 15;
        uint64_t acc = 0;
        if (l < kb && k >= 1 && k - 1 < nrest) {
            const uint64_t lv = F.linv[l];
#pragma unroll
            for (int g = 0; g < 16; ++g) acc ^= S.t16[((g << 4) | static_cast<int>((lv >> (4 * g)) & 15u)) * 15 + k - 1];
        }
        S.U[i] = acc;
        if (k >= 1) pk->u[l][k - 1] = acc;
    }
    // in the same phase (nothing here feeds the solve): the carry finalize tables from the
    // basis and the packet's L11^-1 rows (the lmap is a worker's job)
    for (int i = tid; i < 8 * 256; i += kPT) {
        const int g = i >> 8, v = i & 255;
        uint64_t f = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if ((v >> b) & 1) f ^= F.fbas[8 * g + b];
        S.F[i] = f;
    }
    if (tid >= 960) pk->linv[tid - 960] = F.linv[tid - 960];
    if (tid == 0) pk->leaf = leaf;
    F2_CLK(if (clk) st->dbg[26] = clock64() - c0;)
    F2_STAMP(st, 21);
    const int mv0 = first ? 0 : static_cast<int>(st->nmoved);
    const int64_t pkb = first ? 0 : st->panel_kb;
    int moved = 0, off = 0;
    if (warp < 4) {
        const int sl = tid;
        moved = sl < span && F.src[sl] != sl;
        const unsigned bm = __ballot_sync(FULL_MASK, moved);
        off = __popc(bm & ((1u << lane) - 1));
        if (lane == 0) F.wcount[warp] = __popc(bm);
    }
    for (int l = tid; l < kb; l += kPT) {
        P[base + l] = base + F.step_p[l];
        Qp[base + l] = qcol_off + wl * 64 + F.step_c[l];
        st->panel_q[pkb + l] = leaf * 64 + F.step_c[l];
        st->brow[leaf * 64 + F.step_c[l]] = base + l;
    }
    __syncthreads();
    F2_CLK(if (clk) st->dbg[27] = clock64() - c0;)
    F2_STAMP(st, 22);
    // pivot rows' slices: earlier leaf words as carried, the final leaf word, U
    for (int i = tid; i < kb * 16; i += kPT) {
        const int l = i >> 4, k = i & 15;
        if (k >= nwp) continue;
        const int ss = F.src[l];
        const uint64_t v = k < leaf ? S.win[pb][ss][k] : (k == leaf ? F.uf[l] : S.U[l * 16 + k - leaf]);
        A.w[Z.wphys[pb][ss] * stride + pw0 + k] = v;
    }
    if (warp < 4 && moved) {
        int o = off;
        for (int w2 = 0; w2 < warp; ++w2) o += F.wcount[w2];
        pmap[base + tid] = Z.wphys[pb][F.src[tid]];
        st->moved[mv0 + o] = base + tid;
    }
    if (tid < kPW) Z.srcprev[tid] = F.src[tid];
    // carry tables T[g4][e] over the solved rows (word index relative to the leaf word)
    {
        const int g4 = tid >> 6, e = (tid >> 2) & 15, wq = tid & 3;
        uint64_t v[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = F.posc[4 * g4 + b];
            if (((e >> b) & 1) && r >= 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] ^= S.U[r * 16 + 4 * wq + k];
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) S.T[(g4 * 16 + e) * kW + 4 * wq + k] = v[k];
    }
    if (warp == 0) {
        uint64_t mk = 0;
        for (int l = lane; l < kb; l += 32) mk |= 1ull << F.step_c[l];
        mk = warp_or64(mk);
        int nm = 0, hi = -1;
        for (int w2 = 0; w2 < 4; ++w2) nm += F.wcount[w2];
        for (int w2 = 3; w2 >= 0 && hi < 0; --w2)
            if (F.wcount[w2]) hi = w2;
        if (lane == 0) {
            st->leaf_mask = mk;
            st->nmoved = mv0 + nm;
            const int64_t h = hi < 0 ? 0 : base + 32 * (hi + 1);
            const int64_t prev = first ? 0 : st->pmap_hi;
            const int64_t ph = h > prev ? h : prev;
            st->pmap_hi = ph;
            st->leaf_r = base;
            st->leaf_kb = kb;
            st->r = base + kb;
            if (first) st->panel_r = base;
            st->panel_kb = pkb + kb;
            pk->r0 = base;
            pk->kb = kb;
            pk->lo = base + kb + kPW;
            pk->pmap_hi = ph;
        }
    }
    __syncthreads();
    F2_CLK(if (clk) st->dbg[21] = clock64() - c0;)
    return kb;
}

}  // namespace

__global__ void __launch_bounds__(kPT, 1)
k_panel_pipe(Mat A, int64_t pw0, int width, int64_t pw1, PlsState* st, int64_t* P, int64_t* Qp, int64_t* pmap,
             int64_t qcol_off, unsigned* bar) {
    extern __shared__ __align__(16) uint64_t dsm[];
    __shared__ LeafInfo L;
    __shared__ PipeStatic Z;
    __shared__ int64_t s_ctl[4];
    PipeSmem& S = *reinterpret_cast<PipeSmem*>(dsm);
    uint64_t* tab = dsm;  // workers / fallback: T4 or the 8-bit solve table
    uint64_t* X = tab + kTab;
    uint64_t* Fw = X + 64 * kW;
    const int nleaves = (width + 63) / 64;
    const int nwp = static_cast<int>(pw1 - pw0);
    unsigned target = 0;
#ifdef F2_TIMELINE
    if (threadIdx.x == 0) atomicMin(&st->tl[0][(pw0 / 16) & 127], gtimer());
#endif
    // Every row is a pivot already (a wide matrix past its row rank): the panel has nothing to
    // pivot or update.  Every CTA sees the same r (final since the previous panel's kernel) and
    // leaves at once; CTA 0 publishes the empty panel for the gather / TRSM / Schur launches.
    if (ldi(&st->r) >= A.m) {
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < nleaves * 64; i += kPT) st->brow[i] = -1;
            if (threadIdx.x == 0) {
                const int64_t r = ldi(&st->r);
                st->leaf_mask = 0;
                st->nmoved = 0;
                st->pmap_hi = 0;
                st->leaf_r = r;
                st->leaf_kb = 0;
                st->panel_r = r;
                st->panel_kb = 0;
            }
        }
        return;
    }
    int kbprev = 0, pkc = 0;  // CTA 0's carry state (uniform across its threads)
    // Rank-deficient / sparse panels: after a leaf needed the general search (st->hint), each
    // fresh window has the idle workers check whether any row past it is nonzero in the
    // panel's remaining words (bar[1]: scans done, bar[2]: last nonzero scan + 1).  All zero:
    // those rows can never hold a candidate nor be touched by a pivot for the rest of the
    // panel, so the window decides every column (past_zero, sticky) -- a zero column no
    // longer sends the leaf to the general search.
    bool past_zero = false;
    // (CTA 0) the 96-slot pivot search could not decide a leaf of this panel, or an earlier
    // panel needed the general search (rank-deficient / sparse input): search all 128 slots
    bool search4 = __ldcg(&st->hint) != 0;
    unsigned nscan = 0;
    __shared__ int s_pz;
    int64_t state = S_FRESH, leaf = 0, wpk = -1, wleaf = 0;
    for (int it = 0;; ++it) {
        if (it > 0) {
            if (threadIdx.x < 4) s_ctl[threadIdx.x] = ldi(&st->ctl[it & 1][threadIdx.x]);
            __syncthreads();
            state = s_ctl[0];
            leaf = s_ctl[1];
            wpk = s_ctl[2];
            wleaf = s_ctl[3];
            __syncthreads();
        }
        // (clocks build) CTA 0's iteration starts of a late panel (panel 56 of a 64-panel run)
        F2_CLK(if (pw0 == 16 * 56 && blockIdx.x == 0 && threadIdx.x == 0 && it < 24) st->prof[32 + it] = clock64();)
        F2_CLK(const bool lclk = pw0 == 16 * 56 && blockIdx.x == 0 && threadIdx.x == 0 && it == 5;)
        F2_CLK(if (lclk) st->dbg[1] = clock64();)  // control word read
        if (state == S_DONE) break;
#ifdef F2_PANEL_PROFILE
        if (threadIdx.x == 0 && blockIdx.x == 0) g_prof_on = (pw0 == 0 && leaf == 2 && state == S_CARRY);
        __syncthreads();
#endif
        F2_STAMP(st, 0);
        const bool scan = state == S_FRESH && __ldcg(&st->hint) != 0;  // (the same in every CTA)
        if (scan) ++nscan;
        if (blockIdx.x == 0) {
            int64_t nstate = S_DONE, nleaf = leaf, nwpk = -1, nwleaf = 0;
            const int j = static_cast<int>(leaf);
            const int pb = j & 1;
            if (scan) {
                if (!past_zero) {
                    if (threadIdx.x == 0) {
                        const unsigned want = nscan * (gridDim.x - 1);
                        unsigned v;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar + 1) : "memory");
                        } while (v < want);
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar + 2) : "memory");
                        s_pz = v < nscan;
                    }
                    __syncthreads();
                    past_zero = s_pz != 0;
                }
            }
            if (state == S_FRESH || state == S_CARRY || state == S_FINAL) {
                F2_CLK(const long long cb = clock64();)
                pipe_build_window(A, pw0, nwp, pmap, st, S, Z, pb, state != S_FRESH, kbprev, j - 1,
                                  j == 0 ? 0 : st->pmap_hi, state == S_FINAL);
                F2_CLK(if (pw0 == 0 && j == 2 && threadIdx.x == 0) st->dbg[22] = clock64() - cb;)
                F2_CLK(if (lclk) st->dbg[2] = clock64();)  // window built
                F2_STAMP(st, 1);
                if (state == S_FINAL) {
                    pipe_write_back(A, pw0, nwp, S, Z, pb);
                    nstate = S_DONE;
                } else {
                    const int lw = width - 64 * j < 64 ? width - 64 * j : 64;
                    PlsState::Packet* pk = &st->pk[pkc & 1];
                    const int kb = pipe_fast_leaf(A, pw0, nwp, j, lw, st, P, Qp, pmap, qcol_off, S, Z, pb, pk, nleaves,
                                                  state == S_CARRY, past_zero, search4);
                    F2_CLK(if (lclk) st->dbg[3] = clock64();)  // leaf done
                    F2_STAMP(st, 2);
                    if (kb >= 0) {
                        kbprev = kb;
                        nwpk = pkc & 1;
                        nwleaf = j;
                        ++pkc;
                        nstate = j + 1 < nleaves ? S_CARRY : S_FINAL;
                        nleaf = j + 1;
                        // every row is a pivot (r = m, e.g. a wide matrix past its rank): the
                        // remaining leaves have no rows to pivot or update -- straight to the
                        // final step (the workers still take this leaf's packet: CTA 1 builds
                        // its TRSM map there), so the empty panels after full row rank cost
                        // one leaf instead of sixteen
                        if (st->r >= A.m) nstate = S_FINAL;
                        // a leaf without pivots while no row past the window is nonzero in the
                        // panel's remaining words (past_zero): if the window's remaining words
                        // are zero too, no column of this panel can hold another pivot -- the
                        // rank-deficient panels past the rank cost one or two leaves, not sixteen
                        if (nstate == S_CARRY && kb == 0 && past_zero) {
                            uint64_t acc = 0;
                            for (int i = threadIdx.x; i < kPW * 16; i += kPT) {
                                const int k = i & 15;
                                if (k > j && k < nwp) acc |= S.win[pb][i >> 4][k];
                            }
                            if (!__syncthreads_or(acc != 0)) nstate = S_FINAL;
                        }
                    } else {  // undecidable in the window: hand the window back, search globally
                        pipe_write_back(A, pw0, nwp, S, Z, pb);
                        nstate = S_GENERAL;
                        nleaf = j;
                    }
                }
            } else if (state == S_GENERAL) {
                const int lw = width - 64 * j < 64 ? width - 64 * j : 64;
                if (threadIdx.x == 0) st->hint = 1;
                // (the window is written back: its SMEM holds the search's compact row list)
                leaf_pivot_body(A, pw0 + j, lw, j == 0, j, nleaves * 64, st, P, Qp, pmap, qcol_off,
                                reinterpret_cast<uint8_t*>(dsm), static_cast<int>(kPipeSmem / 17) & ~63);
                __syncthreads();
                load_leaf(st, L);
                if (threadIdx.x < 64) st->fbasis[threadIdx.x] = L.fb[threadIdx.x];
                leaf_lmap(st, L, j, X);
                solve_pivot_rows(A, pw0 + j + 1, pw1, pmap, L, X, tab, st);
                publish_from_state(st, &st->pk[pkc & 1]);
                nwpk = pkc & 1;
                nwleaf = j;
                ++pkc;
                nstate = S_IDLE;
                nleaf = j + 1;
            } else if (state == S_IDLE) {
                nstate = j < nleaves ? S_FRESH : S_DONE;
                nleaf = j;
            }
            __syncthreads();
            if (threadIdx.x == 0) {  // read by every CTA after the barrier (parity: a late
                int64_t* c = st->ctl[(it + 1) & 1];  // reader of this iteration's word is never overtaken)
                c[0] = nstate;
                c[1] = nleaf;
                c[2] = nwpk;
                c[3] = nwleaf;
            }
        } else if (scan) {  // a fresh window: is any row past it nonzero in the remaining words?
            const int j = static_cast<int>(leaf);
            const int64_t lo = ldi(&st->r) + kPW;
            const int nwr = nwp - j, k = threadIdx.x & 15;
            uint64_t acc = 0;
            for (int64_t pos = lo + (blockIdx.x - 1) * (kPT / 16) + (threadIdx.x >> 4); pos < A.m;
                 pos += static_cast<int64_t>(gridDim.x - 1) * (kPT / 16))
                if (k < nwr) acc |= ldw(A.w + ldi(pmap + pos) * A.stride + pw0 + j + k);
            if (__syncthreads_or(acc != 0) && threadIdx.x == 0) atomicMax(bar + 2, nscan);
            if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar + 1) : "memory");
        } else if (wpk >= 0) {
            const PlsState::Packet* pk = &st->pk[wpk];
            if (blockIdx.x == 1 && s_ctl[0] != S_IDLE) pipe_worker_lmap(st, pk, X);
            if (ldi(&pk->kb) != 0) {
                worker_prep(pk, L, X, Fw, tab);
                const int64_t rows = A.m - L.lo;
                const int ntiles = rows > 0 ? static_cast<int>((rows + kRows - 1) / kRows) : 0;
                for (int ty = blockIdx.x - 1; ty < ntiles; ty += gridDim.x - 1)
                    update_tile(A, pw0 + wleaf, pw1, pmap, L, ty, Fw, tab, st);
            }
        }
        F2_STAMP(st, 3);
#ifdef F2_PANEL_PROFILE
        if (threadIdx.x == 0 && blockIdx.x == 0) g_prof_on = 0;
#endif
        F2_CLK(const long long cbar = clock64();)
        F2_CLK(if (lclk) st->dbg[4] = cbar;)  // at the grid barrier
        grid_barrier(bar, target);
        F2_CLK(if (lclk) st->dbg[5] = clock64();)  // barrier passed
        F2_CLK(if (pw0 == 0 && leaf == 2 && threadIdx.x == 0 && blockIdx.x == 0) st->dbg[23] = clock64() - cbar;)
        F2_CLK(if (pw0 == 0 && leaf == 2 && threadIdx.x == 0 && blockIdx.x == 1) st->dbg[24] = clock64() - cbar;)
    }
#ifdef F2_TIMELINE
    if (threadIdx.x == 0) atomicMax(&st->tl[1][(pw0 / 16) & 127], gtimer());
#endif
}

void launch_panel_pipe(cudaStream_t s, const Mat& A, int64_t pw0, int width, int64_t pw1, PlsState* st, int64_t* P,
                       int64_t* Qp, int64_t* pmap, int64_t qcol_off, unsigned* bar, int nsm, bool cooperative) {
    // Non-cooperative launches (the look-ahead side stream, next to a running Schur
    // update) rely on every CTA becoming resident eventually: the only other work on
    // the device is the Schur kernel, whose CTAs never wait, and the grid (<= SMs)
    // fits one CTA per SM.
    cudaMemsetAsync(bar, 0, 4 * sizeof(unsigned), s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nsm));
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = kPipeSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = cooperative ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_panel_pipe, A, pw0, width, pw1, st, P, Qp, pmap, qcol_off, bar);
}


void setup_panel_kernels() {
    cudaFuncSetAttribute(k_panel_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kPipeSmem));
}

}  // namespace f2g
