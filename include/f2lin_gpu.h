/*
 * f2lin_gpu.h — C-ABI drop-in surface of the B200 GF(2) PLS engine.
 *
 * Every entry point below replaces one entry point of the reference C++ API
 * (`f2lin`, /root/reference/proj/include/f2lin/*.hpp); the cited file:line is
 * the interface it stands in for.  Argument meaning and error behaviour mirror
 * the reference: each `std::invalid_argument` becomes F2_INVALID_ARGUMENT, each
 * `std::out_of_range` becomes F2_OUT_OF_RANGE, and outputs are written only on
 * the paths where the reference would have written them.
 *
 * Conventions
 *  - A matrix lives in HBM (`f2_matrix`), bit-packed row-major in 64-bit words,
 *    bit j of a row in word j/64 at position j%64 (bitmat.hpp:3-6).  Device rows
 *    are padded to a multiple of 16 words (128 B); padding bits are zero.
 *  - Host word arrays passed to upload/download and to the *_host entry points
 *    use any row stride >= ceil(ncols/64) words (the reference uses exactly that).
 *  - Permutations are LAPACK-style transposition vectors of uint64_t, the width
 *    of the reference's std::size_t (perm.hpp:3-7).
 *  - Windows are half-open row/column bounds (MatrixWindow, bitmat.hpp:239-250).
 *  - Calls are synchronous on return and stream-ordered on the library's stream.
 *  - There is no CPU fallback: without a CUDA device every compute entry point
 *    returns F2_NO_DEVICE.
 */
#ifndef F2LIN_GPU_H
#define F2LIN_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum f2_status {
    F2_OK = 0,
    F2_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    F2_OUT_OF_RANGE = 2,     /* std::out_of_range in the reference      */
    F2_CUDA_ERROR = 3,
    F2_NO_DEVICE = 4,
    F2_OUT_OF_MEMORY = 5,
    F2_FORMAT_ERROR = 6      /* io::FormatError in the reference            */
};

/* enum class Algorithm — pls.hpp:18 */
enum f2_algorithm { F2_ALG_GAUSS = 0, F2_ALG_M4RI = 1, F2_ALG_MMPF = 2, F2_ALG_PLS = 3, F2_ALG_HYBRID = 4 };

/* struct EliminationConfig — pls.hpp:26-35 (0 = automatic, as in the reference) */
typedef struct f2_elim_config {
    unsigned k;
    uint64_t cutoff_bytes;
    double hybrid_threshold;
    int algorithm;
} f2_elim_config;

/* MatrixWindow bounds — bitmat.hpp:239-250 (r_start, c_start, r_end, c_end) */
typedef struct f2_window {
    size_t r0, c0, r1, c1;
} f2_window;

/* class BitMatrix — bitmat.hpp:90-234, resident in HBM */
typedef struct f2_matrix f2_matrix;

/* ---- library / device ------------------------------------------------- */
const char* f2_last_error(void);
int f2_device_count(void);
int f2_set_device(int device);

/* ---- BitMatrix lifecycle (bitmat.hpp:94-140) ---------------------------- */
int f2_matrix_create(size_t nrows, size_t ncols, f2_matrix** out);      /* BitMatrix(m,n), zeroed   */
void f2_matrix_destroy(f2_matrix* a);                                    /* ~BitMatrix               */
size_t f2_matrix_nrows(const f2_matrix* a);                              /* nrows()  bitmat.hpp:142  */
size_t f2_matrix_ncols(const f2_matrix* a);                              /* ncols()  bitmat.hpp:143  */
size_t f2_matrix_stride(const f2_matrix* a);                             /* device row stride, words */
uint64_t* f2_matrix_device_ptr(f2_matrix* a);                            /* raw HBM words            */
int f2_matrix_upload(f2_matrix* a, const uint64_t* host, size_t host_stride_words);
int f2_matrix_download(const f2_matrix* a, uint64_t* host, size_t host_stride_words);
int f2_matrix_copy(f2_matrix* dst, const f2_matrix* src);               /* BitMatrix copy (deep)    */
int f2_matrix_clear(f2_matrix* a);                                       /* clear()  bitmat.hpp:207  */
/* BitMatrix::randomize — bitmat.hpp:196, bitmat.cpp:136-154: same SplitMix64
 * stream, bit for bit, generated on the device (counter-based). */
int f2_matrix_randomize(f2_matrix* a, double density, uint64_t seed);
/* config 5's fixed-weight sparse rows (the reference has no generator):
 * one SplitMix64 stream (prng.hpp:11-22), per row draws next() % ncols, repeats rejected */
int f2_matrix_fixed_weight(f2_matrix* a, size_t weight, uint64_t seed);
/* order-sensitive fingerprint over the reference packing (tests/oracle_lib.digest) */
int f2_matrix_digest(const f2_matrix* a, uint64_t* out);

/* pinned host memory for the end-to-end path */
void* f2_host_alloc(size_t bytes);
void f2_host_free(void* p);

/* ---- PLS decomposition ------------------------------------------------- */
/* std::size_t mmpf_pls(MatrixWindow a, span<size_t> p, span<size_t> q, unsigned k=0)
 *   — mmpf.hpp:35-36, mmpf.cpp:81-121.  p has w.r1-w.r0 entries, q has w.c1-w.c0. */
int f2_mmpf_pls(f2_matrix* a, f2_window w, uint64_t* p, size_t plen, uint64_t* q, size_t qlen,
                unsigned k, uint64_t* rank);
/* std::size_t pls_recursive(MatrixWindow, span p, span q, const EliminationConfig&)
 *   — pls.hpp:42-43, pls.cpp:105-113.  cfg may be NULL (= {}). */
int f2_pls_recursive(f2_matrix* a, f2_window w, uint64_t* p, size_t plen, uint64_t* q, size_t qlen,
                     const f2_elim_config* cfg, uint64_t* rank);
/* Host-buffer variants (the call a caller holding a host BitMatrix makes):
 * upload, decompose, download in one call.  `words` is updated in place. */
int f2_mmpf_pls_host(uint64_t* words, size_t nrows, size_t ncols, size_t stride_words, uint64_t* p,
                     uint64_t* q, unsigned k, uint64_t* rank);
int f2_pls_recursive_host(uint64_t* words, size_t nrows, size_t ncols, size_t stride_words, uint64_t* p,
                          uint64_t* q, const f2_elim_config* cfg, uint64_t* rank);

/* std::size_t default_cutoff_bytes() — pls.cpp:37-53 (host CPU L2, F2_L2_BYTES) */
uint64_t f2_default_cutoff_bytes(void);
/* detail::auto_table_bits — mul.cpp:9-14 */
unsigned f2_auto_table_bits(size_t dim);

/* void rref_from_pls(MatrixWindow a, size_t rank, span<const size_t> q) — pls.hpp:54, pls.cpp:128-155 */
int f2_rref_from_pls(f2_matrix* a, f2_window w, uint64_t rank, const uint64_t* q, size_t qlen);
/* echelonize: RREF via pls_recursive + rref_from_pls (equals gauss_rref / m4ri_rref, gauss.hpp:28) */
int f2_rref(f2_matrix* a, f2_window w, const f2_elim_config* cfg, uint64_t* rank);
/* size_t m4ri_rref(BitMatrix&, unsigned k = 0, bool full = true) — m4ri.hpp:41, m4ri.cpp:68-87.
 * full: the RREF; !full: M4RI's echelon form (each gauss_submatrix block reduced inside
 * itself, rows above untouched), bit-identical to the reference's.  k > 8 -> F2_INVALID_ARGUMENT */
int f2_m4ri_rref(f2_matrix* a, unsigned k, int full, uint64_t* rank);
/* size_t hybrid_rref(BitMatrix&, const EliminationConfig&) — pls.hpp:61, pls.cpp:163-198 (the RREF) */
int f2_hybrid_rref(f2_matrix* a, const f2_elim_config* cfg, uint64_t* rank);
/* size_t rank(const BitMatrix&, const EliminationConfig&) — pls.hpp:64, pls.cpp:200-216 (A untouched) */
int f2_rank(const f2_matrix* a, const f2_elim_config* cfg, uint64_t* rank);

/* ---- multiply / triangular solve --------------------------------------- */
/* void addmul(MatrixWindow c, MatrixWindow a, MatrixWindow b, unsigned k=0) — mul.hpp:20, mul.cpp:102-107 */
int f2_addmul(f2_matrix* c, f2_window wc, f2_matrix* a, f2_window wa, f2_matrix* b, f2_window wb,
              unsigned k);
/* BitMatrix mul_m4rm(const BitMatrix&, const BitMatrix&, unsigned k=0) — mul.hpp:17, mul.cpp:90-100.
 * *out is created by the call. */
int f2_mul_m4rm(const f2_matrix* a, const f2_matrix* b, unsigned k, f2_matrix** out);
/* void trsm_lower_left_unit(MatrixWindow l, MatrixWindow b) — mul.hpp:24, mul.cpp:109-131 */
int f2_trsm_lower_left_unit(f2_matrix* l, f2_window wl, f2_matrix* b, f2_window wb);
/* void trsm_upper_left_unit(MatrixWindow u, MatrixWindow b) — mul.hpp:28, mul.cpp:133-155 */
int f2_trsm_upper_left_unit(f2_matrix* u, f2_window wu, f2_matrix* b, f2_window wb);
/* void compress_columns(BitMatrix&, rank, const Permutation& q) — perm.hpp:61, perm.cpp:55-60 */
int f2_compress_columns(f2_matrix* a, uint64_t rank, const uint64_t* q, size_t qlen);
/* Permutation::apply_rows / apply_rows_inverse — perm.hpp:42-45, perm.cpp:29-38 */
int f2_apply_rows(f2_matrix* a, f2_window w, const uint64_t* p, size_t plen, int inverse);

/* ---- column-sharded PLS (one rank per GPU; paper_1006_1744_b200/dist.py) ----
 * The reference has no distributed entry point: this is the multi-GPU form of
 * pls_recursive (pls.hpp:42-47, the recursion pls.cpp:63-103 split by columns,
 * SURVEY.md §8e).  Rank k holds panels k, k+N, ... of W bits side by side in a
 * local matrix with all m rows.  Every call ENQUEUES on the caller's CUDA streams
 * (cudaStream_t passed as void*) and returns without waiting on the GPU.
 * Exchange buffer of one panel: f2_dist_buffer_words(m, W) words = the panel's
 * words of every row (W/64 per row) then its header; a broadcast may start at
 * row r_lo <= the panel's first pivot row (its tail is all a receiver reads).
 *   f2_dist_begin    reset the elimination state (r = 0, identity row order)
 *   f2_dist_factor   owner of a panel: pivot search + panel update, export into buf
 *   f2_dist_step     every rank, panel p: import (owner = 0), row gather, TRSM and
 *                    Schur update of the local trailing columns (from word tw0); with
 *                    lookahead = 1 (this rank owns panel p+1, whose local words start
 *                    at tw0) the next panel's columns are updated first and
 *                    f2_dist_factor(p+1) runs on side_stream beside the rest
 *   f2_dist_note     record (kb, panel_r) of buf's header on `stream`;
 *   f2_dist_header_rk  wait for that record and return it
 *   f2_dist_finish   rank, P (m entries) and the pivot columns (Q prefix) */
size_t f2_dist_buffer_words(size_t nrows, unsigned panel_bits);
int f2_dist_begin(f2_matrix* a, unsigned panel_bits, size_t npanels, void* stream);
int f2_dist_factor(f2_matrix* a, size_t pw0, unsigned width_bits, uint64_t panel_col, uint64_t* buf, int ctas,
                   void* stream);
int f2_dist_step(f2_matrix* a, int64_t p, int owner, size_t pw0, unsigned width_bits, const uint64_t* buf,
                 size_t tw0, int lookahead, unsigned next_width, uint64_t next_col, uint64_t* next_buf, int side_ctas,
                 void* main_stream, void* side_stream);
int f2_dist_note(const uint64_t* buf, int64_t p, void* stream);
int f2_dist_header_rk(int64_t p, uint64_t* kb, uint64_t* r0);
int f2_dist_finish(f2_matrix* a, void* stream, uint64_t* rank, uint64_t* p, size_t plen, uint64_t* pivcols,
                   size_t qcap);
/* a non-owning f2_matrix over caller device memory (stride a multiple of 16 words);
 * f2_matrix_destroy releases only the handle */
int f2_matrix_view(uint64_t* dev, size_t nrows, size_t ncols, size_t stride_words, f2_matrix** out);
/* compress_columns of a packed PLS result from its pivot columns (perm.cpp:18-21) */
int f2_pls_compress(f2_matrix* a, uint64_t rank, const uint64_t* pivcols);
/* pls_recursive's full Q (tail included) from (m, n, cutoff, pivot columns) — pls.cpp:63-103 */
int f2_recursive_q(size_t m, size_t n, uint64_t cutoff, uint64_t rank, const uint64_t* pivcols, uint64_t* q);

/* ---- on-disk formats (io.hpp:3-11, io.cpp) ------------------------------ */
enum f2_format { F2_FMT_ASCII = 0, F2_FMT_BINARY = 1 }; /* io::Format (io.hpp:22) */
/* header only: dimensions and the sniffed format (io.cpp:118-126) */
int f2_io_probe(const char* path, uint64_t* nrows, uint64_t* ncols, int* format);
/* io::read_matrix(path) into a host buffer of the probed shape (any row stride >= ceil(n/64)) */
int f2_io_read_host(const char* path, uint64_t* words, size_t stride_words, uint64_t nrows, uint64_t ncols);
/* io::write_matrix(path, a, fmt) from a host buffer */
int f2_io_write_host(const char* path, const uint64_t* words, size_t stride_words, uint64_t nrows, uint64_t ncols,
                     int format);
/* io::read_matrix(path, &detected) straight into HBM (pinned double-buffered stream) */
int f2_matrix_load(const char* path, f2_matrix** out, int* detected);
/* io::write_matrix(path, a, fmt) straight from HBM */
int f2_matrix_store(const f2_matrix* a, const char* path, int format);
/* io::write_permutation / read_permutation (io.cpp:135-160); *len always set, entries copied when len <= cap */
int f2_write_permutation(const char* path, const uint64_t* p, size_t len);
int f2_read_permutation(const char* path, uint64_t* p, size_t cap, size_t* len);

/* ---- instrumentation (bench.py roofline) -------------------------------- */
/* When enabled, the library brackets every launch of kernel family `kind`
 * with CUDA events on its own stream and accumulates launches, device ms and
 * the launch's algorithmic work (bytes for the table-apply, bit-ops for the
 * multiply).  kind: 0 = table-apply/M4RM multiply, 1 = leaf pivot search,
 * 2 = pivot-row TRSM, 3 = everything else. */
int f2_stats_enable(int enable);
int f2_stats_get(int kind, uint64_t* launches, double* ms, double* bytes, double* bitops);
int f2_stats_reset(void);
/* CUDA-event timer on the library's stream (start/stop bracket device work) */
int f2_timer_start(void);
int f2_timer_stop(double* ms);
/* kernel launches issued by the last compute call (all families) */
uint64_t f2_last_launch_count(void);
/* kernel nodes of the CUDA graph the last graph-replayed PLS launched (0: not a graph run) */
uint64_t f2_last_graph_kernels(void);
/* phase clocks of the last leaf (only builds compiled with -DF2_LEAF_PROFILE fill them) */
int f2_debug_clocks(long long* out, int n);
/* globaltimer stamps of the panel kernel (only builds compiled with -DF2_PANEL_PROFILE fill them) */
int f2_debug_prof(long long* out, int n);
/* per-panel start/end stamps of the panel kernel and the Schur (only -DF2_TIMELINE builds fill them) */
int f2_debug_timeline(unsigned long long* out, int n);
/* engine tuning (panel width in bits for pls_recursive; 0 = default) */
int f2_set_panel_bits(unsigned bits);

#ifdef __cplusplus
}
#endif
#endif /* F2LIN_GPU_H */
