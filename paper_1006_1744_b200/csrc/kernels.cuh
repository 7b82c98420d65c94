// Host-side launchers of the engine's kernels (one per .cu translation unit).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "f2gpu.cuh"

namespace f2g {

// kernel launch with programmatic stream serialization (the kernel must call pdl_wait()
// first); F2_NO_PDL=1 falls back to ordinary launches
extern bool g_pdl;
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    if (!g_pdl) {
        kernel<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// leaf.cu
// the panel's row gather; with snap != nullptr the same launch also takes the panel's
// snapshot (kSnap* below) from Cf's words coef_w0.. (Cf == A: read through pmap)
void launch_perm(cudaStream_t s, const Mat& A, int64_t nwords, const PlsState* st, int64_t* pmap, uint64_t* scratch,
                 int64_t* snap = nullptr, int nleaves = 0, const Mat* Cf = nullptr, int64_t coef_w0 = 0,
                 int64_t* plan = nullptr);
// plan (1 + 2 * kMaxMoved words): the gather's {count, (destination, source) rows...}, so
// launch_plan_perm can repeat it later on words [w0, w1) (w0 even: 16-byte accesses)
constexpr int64_t kPlanWords = 1 + 2 * static_cast<int64_t>(kMaxMoved);
void launch_plan_perm(cudaStream_t s, const Mat& A, int64_t w0, int64_t w1, const int64_t* plan, uint64_t* scratch);
void launch_pmap_init(cudaStream_t s, int64_t* pmap, int64_t m);
void launch_panel_lmaps(cudaStream_t s, const Mat& Cf, int64_t pw0, int nleaves, PlsState* st);
constexpr int64_t dist_header_words(int W) { return 4 + 2 * static_cast<int64_t>(W) + 2 * kMaxMoved; }
void launch_dist_export(cudaStream_t s, const Mat& A, int64_t pw0, int nwp, const PlsState* st, const int64_t* pmap,
                        const int64_t* P, uint64_t* buf, int W, int64_t col, int nsm);
void launch_dist_import(cudaStream_t s, PlsState* st, int64_t* pmap, int64_t* P, int64_t* Qp, const int64_t* hdr,
                        int W);
void setup_leaf_kernels();


// trsm.cu — forward substitution of pivot rows by 8-column groups with
// Gray tables (the M4RI-style TRSM of mul.cpp:109-131, blocked for SMEM).
struct PivotSet {
    int mode;              // 0: leaf (st->q, leaf_r, leaf_kb); 1: panel (st->panel_q, panel_r, panel_kb);
                           // 2: static identity pivots (q_t = t, r0, kb given)
    int64_t r0, kb;        // used by mode 2
};
void launch_pivot_trsm(cudaStream_t s, const Mat& A, int64_t coef_w0, int coef_words, int64_t tw0,
                       int64_t tw1, const PlsState* st, PivotSet ps, const Mat* L);
void launch_panel_trsm(cudaStream_t s, const Mat& A, const Mat& Cf, int64_t coef_w0, int nleaves, int64_t tw0,
                       int64_t tw1, const PlsState* st);
void setup_trsm_kernels();

// m4rm.cu — C ^= A * B by 8-bit Gray tables in SMEM (M4RM, mul.cpp:21-68),
// also the MMPF table-apply (m4ri.cpp:28-38) when K = one 64-bit word.
struct TableApply {
    Mat C;                 // rows [c_r0, c_r1), words [cw0, cw1)
    int64_t c_r0, c_r1, cw0, cw1;
    Mat A;                 // coefficient rows: A row = a_r0 + (i - c_r0), words [aw0, aw0+kw)
    int64_t a_r0, aw0;
    int kw;                // coefficient words (K = 64*kw bits, padded with zero bits)
    int64_t kbits;         // valid K bits
    Mat B;                 // B row for raw bit j: brow ? brow[j] : b_r0 + j; B word = bw0 + (cw - cw0)
    int64_t b_r0, bw0;
    const int64_t* brow;
    int row_mode;          // RowMode: static / after leaf / after panel (c_r0 = a_r0 from state)
    const PlsState* st;
    int64_t row_tile0;     // first 1024-row tile of this launch (set by launch_table_apply)
    const int64_t* rk;     // ROWS_AFTER_PANEL from a snapshot {panel_r, panel_kb} instead of st (look-ahead)
};
// snapshot of a finished panel's row range and raw-column -> pivot-row map, so its Schur
// update can run while the next panel's kernel rewrites the state
// Layout (int64 words): [0] panel_r, [1] panel_kb, brow, q (pivot columns, -1 past kb),
// bstart (first pivot index of each leaf), and per leaf j and pivot index t >= bstart[j]
// the solve word M[j][t] = (row t's leaf-j coefficients, masked below its own pivot in
// leaf j) * L_jj^{-1}, i.e. the combination of leaf j's pivot rows as they are before
// leaf j's solve step that row t adds (the panel lmap applied once, not per TRSM CTA).
// Cf words coef_w0 + j of the gathered rows r0 + t hold the coefficients.
constexpr int64_t kSnapBrow = 2, kSnapQ = kSnapBrow + kMaxPanelBits, kSnapBstart = kSnapQ + kMaxPanelBits,
                  kSnapM = kSnapBstart + kMaxPanelBits / 64 + 8,
                  kSnapWords = kSnapM + static_cast<int64_t>(kMaxPanelBits / 64) * kMaxPanelBits;
// U <- L11^{-1} U on words [tw0, tw1) of the panel's pivot rows, from a snapshot only
// (the next panel's kernel may be rewriting the state); strip = words per CTA (1 or 8)
void launch_panel_trsm_snap(cudaStream_t s, const Mat& A, const int64_t* snap, int nleaves, int64_t tw0, int64_t tw1,
                            int strip);
void launch_table_apply(cudaStream_t s, const TableApply& t, int nsm, int64_t expect_rows = 0);
void setup_m4rm_kernels();
// mmpf_apply.cu -- the HBM-streaming table-apply for K <= 64 (one coefficient word per row)
void launch_mmpf_apply(cudaStream_t s, const TableApply& t, int nsm);
void setup_mmpf_apply_kernels();

// schur_f4.cu -- C ^= A * B over GF(2) with K <= 1024 on the tensor cores (tcgen05
// kind::mxf4, parity of exact fp32 counts): the Schur update of pls_recursive and the
// GEMM of addmul/mul_m4rm/TRSM.  Rows are shifted by d = rk ? rk[0] + rk[1] : 0 (a
// device-side pivot count, so PLS launches need no host sync): C row c_r0 + d + i,
// A row a_r0 + d + i, i < rows_end - d.  B row j is brow ? brow[j] : b_r0 + j (brow
// < 0: zero row); C word cw0 + x pairs with B word bw0 + x.
struct F4Job {
    Mat C;
    int64_t c_r0, cw0, cw1;
    Mat A;
    int64_t a_r0, aw0;
    Mat B;
    int64_t b_r0, bw0;
    const int64_t* brow;
    const int64_t* rk;
    int64_t rows_end;
    int64_t kbits;
};
constexpr int64_t kF4MaxK = 1024;
size_t schur_f4_a_bytes(int64_t rows);
size_t schur_f4_b_bytes(int64_t words);
void launch_schur_f4_expand_a(cudaStream_t s, const F4Job& jb, uint8_t* Ax, int nsm);
// Ax: A expanded by launch_schur_f4_expand_a; Bx: scratch; claim: a work counter
void launch_schur_f4(cudaStream_t s, const F4Job& jb, const uint8_t* Ax, uint8_t* Bx, unsigned* claim, int nsm,
                     unsigned long long* tl = nullptr);
void setup_schur_f4_kernels();

// misc.cu
void launch_randomize(cudaStream_t s, const Mat& A, uint64_t threshold, uint64_t seed);
void launch_digest(cudaStream_t s, const Mat& A, unsigned long long* out);
void launch_extract(cudaStream_t s, const Mat& src, int64_t r0, int64_t c0, const Mat& dst);
void launch_insert(cudaStream_t s, const Mat& dst, int64_t r0, int64_t c0, const Mat& src);
void launch_compress(cudaStream_t s, const Mat& A, int64_t rank, const int64_t* Qp, int nsm);
void launch_gather_rows(cudaStream_t s, const Mat& dst, const Mat& src, const int64_t* rowmap, int64_t nrows,
                        int64_t nwords);
void launch_col_swaps(cudaStream_t s, const Mat& A, int64_t rank, const int64_t* q, int nsm);
void setup_misc_kernels();
// panel.cu: all leaves of a panel in one cooperative persistent kernel
void launch_panel_pipe(cudaStream_t s, const Mat& A, int64_t pw0, int width, int64_t pw1, PlsState* st, int64_t* P,
                       int64_t* Qp, int64_t* pmap, int64_t qcol_off, unsigned* bar, int nsm, bool cooperative = true);
void setup_panel_kernels();
void launch_reverse_square(cudaStream_t s, const Mat& dst, const Mat& src, int64_t r);
void launch_block_backsub(cudaStream_t s, const Mat& U, const int64_t* bstart, const int64_t* Qp, int64_t nblocks,
                          int nsm);
void launch_rref_prepare(cudaStream_t s, const Mat& A, int64_t rank, const int64_t* Qp);
void launch_rref_coeffs(cudaStream_t s, const Mat& S, int64_t rank, const int64_t* Qp, const Mat& Lrev, int nsm);
void setup_rref_kernels();

}  // namespace f2g
