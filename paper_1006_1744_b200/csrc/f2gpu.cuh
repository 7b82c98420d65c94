// Shared device-side definitions of the B200 GF(2) PLS engine.
//
// Layout in HBM: a matrix is row-major, 64-bit words, bit j of a row in word
// j/64 at bit j%64 (the reference packing, proj/include/f2lin/bitmat.hpp:3-6),
// with the row stride padded to a multiple of 16 words (128 B) so every row
// starts on a 128-byte line.  Padding bits and padding words are zero and every
// kernel keeps them zero.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace f2g {

constexpr int kMaxPanelBits = 2048;          // widest outer panel W
constexpr int kWinSlots = 4;                 // leaf search window: 32 lanes x 4 slots
constexpr int kWin = 32 * kWinSlots;         // 128 candidate positions in registers
constexpr int kMaxSwaps = kWin + 64;         // window slots + outside positions
constexpr int kOmapSlots = 128;              // open-addressing map for outside swaps
constexpr int kMaxMoved = 8192;              // positions re-mapped during one panel (<= 32 leaves x 192)

struct Mat {
    uint64_t* w;
    int64_t m, n, stride;  // rows, columns (bits), row stride (words)
};

// Device-resident elimination state.  Every kernel of the engine reads its
// row offsets and pivot counts from here, so the host enqueues a fixed,
// data-independent launch sequence and never synchronises mid-factorisation.
//
// Row order inside a panel is virtual: position x of the current row order lives
// in physical row pmap[x] (a separate device array).  The leaves of a panel only
// rewrite pmap; the panel's row transpositions reach the whole row width in one
// gather when the panel ends (k_perm_save / k_perm_put), so a panel's leaves never
// touch columns right of the panel.
struct PlsState {
    int64_t r;         // next pivot position (= pivots found so far)
    int64_t leaf_r;    // r at the start of the current leaf
    int64_t leaf_kb;   // pivots found by the current leaf
    int64_t panel_r;   // r at the start of the current panel
    int64_t panel_kb;  // pivots found so far in the current panel
    int32_t nmoved;    // positions whose pmap entry changed during the panel
    int32_t hint;      // a leaf needed the general search (this run): fresh windows ask the
                       // workers whether any row past them is nonzero (panel.cu, past_zero)
    int64_t pmap_hi;   // pmap[x] == x for every position x >= pmap_hi (this panel)
    uint64_t leaf_mask;                 // pivot columns within the leaf word
    uint64_t ustrict[64];               // leaf pivot words, bits <= pivot cleared
    uint64_t ufull[64];                 // leaf pivot words (L bits, leading 1, S bits)
    uint64_t lmap[kMaxPanelBits / 64][8][256];  // per leaf of the panel: c -> c * L_leaf^{-1}, bytewise
    int32_t q[64];                      // leaf pivot bit positions (0..63)
    int32_t panel_q[kMaxPanelBits];     // panel pivot columns, relative to the panel
    int64_t brow[kMaxPanelBits];        // panel raw column -> pivot row position, -1 if none
    int64_t moved[kMaxMoved];           // positions with pmap[x] != x (may repeat)
    // what CTA 0 of the panel kernel publishes for the row-tile workers, double
    // buffered so the pipelined schedule can write leaf j's while leaf j-1's is read
    struct Packet {
        int64_t r0, kb, lo, pmap_hi;  // pivots at positions r0..r0+kb; workers update positions >= lo
        int32_t q[64];                // pivot bit positions in the leaf word
        uint64_t fb[64];              // finalize basis
        uint64_t u[64][16];           // solved pivot rows over the rest of the panel (word 0 = leaf word + 1)
        uint64_t linv[64];            // rows of L11^{-1} over pivot indices (pipelined kernel: lmap by a worker)
        int64_t leaf;                 // leaf index within the panel
    } pk[2];
    int64_t ctl[2][4];                  // pipelined panel kernel: control word per iteration parity
    uint64_t uleaf[64][16];             // the current leaf's solved pivot rows over the rest of the panel
    uint64_t fbasis[64];                // the current leaf's finalize basis (see panel.cu)
    long long dbg[32];                  // phase clocks (F2_LEAF_PROFILE builds only)
    long long prof[64];                 // globaltimer stamps (F2_PANEL_PROFILE builds only)
    unsigned long long tl[4][128];      // F2_TIMELINE builds: per panel start/end of the panel kernel and the Schur
};


// Loads of data other CTAs may have written during the same (persistent) kernel go
// through L2 (ld.global.cg): the per-SM L1 is not coherent.
__device__ __forceinline__ uint64_t ldw(const uint64_t* p) {
    return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ int64_t ldi(const int64_t* p) { return __ldcg(reinterpret_cast<const long long*>(p)); }

// phase clocks of the panel kernel (tools/dbgclk.py; builds with -DF2_LEAF_CLOCKS only)
#ifdef F2_LEAF_CLOCKS
#define F2_CLK(...) __VA_ARGS__
#else
#define F2_CLK(...)
#endif

#ifdef F2_PANEL_PROFILE
static __device__ int g_prof_on = 0;
#define F2_STAMP(stp, k)                                                               \
    do {                                                                               \
        if (g_prof_on && threadIdx.x == 0 && blockIdx.x == 0) {                                       \
            unsigned long long t_;                                                     \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            const_cast<PlsState*>(stp)->prof[k] = static_cast<long long>(t_);          \
            const_cast<PlsState*>(stp)->dbg[(k) & 31] = clock64();                     \
        }                                                                              \
    } while (0)
#else
#define F2_STAMP(stp, k) \
    do {                 \
    } while (0)
#endif

// Programmatic dependent launch: a kernel launched with launch_pdl may start while its
// stream predecessor drains; it waits here before touching anything the predecessor
// wrote (a no-op for ordinary launches).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// How a table-apply launch finds its C/A rows (device-side offsets).
enum RowMode : int { ROWS_STATIC = 0, ROWS_AFTER_LEAF = 1, ROWS_AFTER_PANEL = 2 };

}  // namespace f2g
