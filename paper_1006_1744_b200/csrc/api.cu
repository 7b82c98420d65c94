// Host side of the B200 GF(2) PLS engine and its C ABI (include/f2lin_gpu.h).
//
// The engine is a blocked right-looking PLS.  The matrix is walked in panels of
// W columns (64 for the MMPF entry point, 1024 by default for the recursive
// entry point).  Per panel:
//   k_panel_pipe     all 64-column leaves of the panel in one persistent kernel:
//                    exact Gaussian pivot search (gauss.cpp:33-49 rule) on CTA 0,
//                    leaf updates of the panel's rows on the other CTAs; the row
//                    transpositions only re-map the panel's virtual row order
//   k_perm_save/put  the panel's transpositions applied to whole rows (perm.cpp:8-16)
//   k_panel_snapshot the finished panel's pivots + per-row solve words
//   k_panel_trsm_snap panel pivot rows solved over the trailing columns (mul.cpp:109-131)
//   k_schur_f4       Schur complement C ^= L21 * U12 on the tensor cores (mul.cpp:21-68),
//                    k_mmpf_apply / k_table_apply for the narrow (MMPF) panels
// and finally k_compress (compress_columns, perm.cpp:18-21) when Q != identity.
// Every row offset and pivot count lives in device memory (PlsState), so the
// launch sequence is fixed by (m, n, W) alone and the host never waits on the
// GPU until the end of the call.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <unistd.h>

#include "../../include/f2lin_gpu.h"
#include "f2gpu.cuh"
#include "kernels.cuh"

using namespace f2g;

struct f2_matrix {
    size_t m = 0, n = 0, stride = 0;
    uint64_t* d = nullptr;
    int device = 0;
    bool owns = true;  // false: a view over caller memory (f2_matrix_view)
};

namespace {

thread_local std::string g_err;
// one compute call at a time per process (shared stream + workspace); recursive so the
// host-buffer entry points hold it across upload, decomposition and download
std::recursive_mutex g_mu;

// Schedule tuning.  The defaults are the measured best on B200; the
// environment overrides exist for A/B runs, are read once at initialisation, and every
// alternative path they select is exercised by tests/test_gpu_tuning.py.
constexpr int kSnapRing = 16;     // panel snapshots in flight (look-ahead: 2; streamed upload: its panels + 2)
constexpr int kUpGroups = 11;     // column groups of a streamed upload
constexpr int kUpMaxPanels = 14;  // panels factored while the upload runs (<= kSnapRing - 2)

struct Tuning {
    bool lookahead = true;        // F2_NO_LOOKAHEAD=1: panel kernels in stream order, no side stream
    bool f4 = true;               // F2_SCHUR_M4RM=1: Schur update on the SMEM table kernel, not tcgen05
    bool graph = true;            // F2_NO_GRAPH=1: enqueue the launch sequence instead of a cached graph
    bool pdl = true;              // F2_NO_PDL=1: ordinary launches instead of programmatic dependent ones
    bool early_wide_trsm = true;  // F2_NO_EARLY_WIDE_TRSM=1: wide TRSM after the fork in early panels too
    bool split_early = false;     // F2_SPLIT_EARLY=1: early panels move the narrow solve + Schur to the side stream
    int side_ctas = 24;           // F2_SIDE_CTAS: CTAs of the look-ahead panel kernel, early panels
    int side_ctas_late = 48;      // F2_SIDE_CTAS_LATE: late panels (0: as early)
    int late_pct = 38;            // F2_LATE_PCT: first late panel, % of the panels
    int wide_early_pct = 62;      // F2_WIDE_EARLY_PCT: panels (%) whose wide TRSM runs early on aux (-1: late_pct)
    bool tw_join_at_fork = false; // F2_TW_JOIN=1: the next panel's kernel waits for the early wide TRSM
    // panel width of the mmpf_pls entry point: its output is the Gaussian one whatever the
    // blocking, and 1024-column panels are 3-6x faster on dense inputs than the paper's
    // 64-column MMPF schedule (F2_MMPF_PANEL_BITS=64: panel kernel + HBM-streaming table-apply)
    unsigned mmpf_bits = 1024;    // F2_MMPF_PANEL_BITS
    // host-buffer entry points: upload in column groups inside the engine, the first
    // panels factoring while the rest of the matrix is still crossing PCIe
    bool stream_upload = true;    // F2_NO_STREAM_UPLOAD=1: upload everything first
    // its plan (upload_plan): group 0 = up_g0 panels, the rest in up_groups - 1 equal
    // groups; streaming panels 0 .. up_ps - 2, their look-ahead kernels on up_side CTAs
    int up_g0 = 8;                // F2_UP_G0
    int up_ps = 9;                // F2_UP_PS (<= kUpMaxPanels)
    int up_groups = 8;            // F2_UP_GROUPS (<= kUpGroups)
    int up_side = 48;             // F2_UP_SIDE
    bool evtl = false;            // F2_EVTL=1 (no graph): per-panel event timeline on stderr
    bool evtl_sync = false;       // F2_EVTL_SYNC=1: synchronise at every timeline mark

    void load(int nsm) {
        auto flag = [](const char* k) {
            const char* e = std::getenv(k);
            return e && e[0] == '1';
        };
        auto num = [](const char* k, int d) {
            const char* e = std::getenv(k);
            return e ? std::atoi(e) : d;
        };
        lookahead = !flag("F2_NO_LOOKAHEAD");
        f4 = !flag("F2_SCHUR_M4RM");
        graph = !flag("F2_NO_GRAPH");
        pdl = !flag("F2_NO_PDL");
        early_wide_trsm = !flag("F2_NO_EARLY_WIDE_TRSM");
        split_early = flag("F2_SPLIT_EARLY");
        const int sc = num("F2_SIDE_CTAS", side_ctas);
        if (sc >= 2 && sc <= nsm) side_ctas = sc;
        const int sl = num("F2_SIDE_CTAS_LATE", side_ctas_late);
        if (sl == 0 || (sl >= 2 && sl <= nsm)) side_ctas_late = sl;
        late_pct = num("F2_LATE_PCT", late_pct);
        wide_early_pct = num("F2_WIDE_EARLY_PCT", wide_early_pct);
        tw_join_at_fork = flag("F2_TW_JOIN");
        const int mb = num("F2_MMPF_PANEL_BITS", static_cast<int>(mmpf_bits));
        if (mb >= 64 && mb <= 1024 && mb % 64 == 0) mmpf_bits = static_cast<unsigned>(mb);
        stream_upload = !flag("F2_NO_STREAM_UPLOAD");
        up_g0 = std::max(1, num("F2_UP_G0", up_g0));
        up_ps = std::min(kUpMaxPanels, std::max(2, num("F2_UP_PS", up_ps)));
        up_groups = std::min(kUpGroups, std::max(2, num("F2_UP_GROUPS", up_groups)));
        const int us = num("F2_UP_SIDE", up_side);
        if (us >= 2 && us <= nsm) up_side = us;
        evtl = flag("F2_EVTL");
        evtl_sync = flag("F2_EVTL_SYNC");
    }
};
Tuning tune;

struct Ctx {
    bool init = false;
    int device = -1;
    int nsm = 148;
    cudaStream_t stream = nullptr;
    // streamed download of finished pivot rows (host-buffer entry points): when set,
    // the engine copies rows [pW, (p+1)W) to dl_host on dl_stream right after panel
    // p's TRSM -- final there whenever panels 0..p each found W pivots (checked after)
    cudaStream_t dl_stream = nullptr;
    cudaEvent_t dl_ev = nullptr, dl_join = nullptr;
    uint64_t* dl_host = nullptr;
    size_t dl_pitch = 0;    // words
    int64_t dl_done = -1;   // rows [0, dl_done) downloaded by the last engine run
    // engine workspace
    PlsState* st = nullptr;
    int64_t* P = nullptr;
    int64_t* Qp = nullptr;
    int64_t* pmap = nullptr;
    unsigned* bar = nullptr;  // grid barrier counter of k_panel_pipe
    // look-ahead: panel p+1's kernel runs on a high-priority side stream with
    // tune.side_ctas CTAs while the Schur update of panel p covers the columns right of it
    cudaStream_t side = nullptr;
    cudaEvent_t la_fork = nullptr, la_join = nullptr;
    cudaStream_t aux = nullptr;  // look-ahead: A-operand expansion next to the narrow TRSM
    cudaEvent_t ax_fork = nullptr, ax_join = nullptr;
    cudaEvent_t tw_fork = nullptr, tw_join = nullptr;  // wide TRSM beside the narrow one (early panels)
    cudaEvent_t nt_done = nullptr;                     // split schedule: narrow TRSM done (on the side stream)
    int64_t* snap = nullptr;  // [kSnapRing][kSnapWords], panel p in slot p % kSnapRing
    // streamed upload (host-buffer entry points, see enqueue_engine): ul_host set = the
    // engine uploads the matrix itself, column group g on `up` (event up_ev[g]); groups
    // 1.. are updated by the streaming panels on their own low-priority streams grp[g]
    const uint64_t* ul_host = nullptr;
    size_t ul_pitch = 0;  // words
    bool ul_used = false;  // the engine ran with ul_host (else the matrix was never uploaded)
    cudaStream_t up = nullptr;
    cudaStream_t grp[kUpGroups] = {};
    cudaEvent_t up_fork = nullptr, gathered = nullptr;
    cudaEvent_t up_ev[kUpGroups] = {}, grp_ev[kUpGroups] = {};
    int64_t* plans = nullptr;  // [kUpMaxPanels][kPlanWords]
    // tensor-core Schur operands (expanded L21 for every row, expanded U12 column tiles)
    uint8_t* f4_ax = nullptr;
    uint8_t* f4_bx = nullptr;
    unsigned* f4_claim = nullptr;
    size_t cap_f4a = 0, cap_f4b = 0;
    uint64_t* scratch = nullptr;
    size_t cap_m = 0, cap_q = 0, cap_scratch = 0;
    int64_t* h_r = nullptr;  // pinned ring of r snapshots (early exit)
    size_t h_r_cap = 0;
    unsigned long long* d_digest = nullptr;
    // stats
    bool stats = false;
    uint64_t launches = 0;
    uint64_t graph_launches = 0;
    uint64_t graph_kernels = 0, last_kernels = 0;  // kernel nodes of the cached PLS graph
    struct Family {
        uint64_t n = 0;
        double ms = 0, bytes = 0, bitops = 0;
    } fam[4];
    unsigned panel_bits = 1024;
};
Ctx g;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? F2_OUT_OF_MEMORY : F2_CUDA_ERROR;
}

#define CK(x)                                          \
    do {                                               \
        cudaError_t e_ = (x);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
    } while (0)

int ensure_init() {
    if (g.init) return F2_OK;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(F2_NO_DEVICE, "no CUDA device visible (this library has no CPU fallback)");
    }
    if (g.device < 0) g.device = 0;
    CK(cudaSetDevice(g.device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, g.device));
    if (prop.major < 10) return fail(F2_NO_DEVICE, "kernels are built for sm_100a (B200)");
    g.nsm = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g.dl_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g.dl_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g.dl_join, cudaEventDisableTiming));
    CK(cudaMalloc(&g.st, sizeof(PlsState)));
    CK(cudaMalloc(&g.d_digest, sizeof(unsigned long long)));
    tune.load(g.nsm);
    g_pdl = tune.pdl;
    setup_leaf_kernels();
    setup_trsm_kernels();
    setup_m4rm_kernels();
    setup_mmpf_apply_kernels();
    setup_schur_f4_kernels();
    setup_misc_kernels();
    setup_rref_kernels();
    setup_panel_kernels();
    CK(cudaMalloc(&g.bar, 4 * sizeof(unsigned)));  // barrier, fresh-window scans (panel.cu)
    {
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&g.side, cudaStreamNonBlocking, hi));
        CK(cudaEventCreateWithFlags(&g.la_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g.la_join, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&g.aux, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&g.ax_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g.ax_join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g.tw_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g.tw_join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g.nt_done, cudaEventDisableTiming));
        CK(cudaMalloc(&g.snap, sizeof(int64_t) * kSnapRing * kSnapWords));
        CK(cudaStreamCreateWithFlags(&g.up, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&g.up_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g.gathered, cudaEventDisableTiming));
        for (int i = 0; i < kUpGroups; ++i) {
            CK(cudaStreamCreateWithPriority(&g.grp[i], cudaStreamNonBlocking, lo));
            CK(cudaEventCreateWithFlags(&g.up_ev[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&g.grp_ev[i], cudaEventDisableTiming));
        }
        CK(cudaMalloc(&g.plans, sizeof(int64_t) * kUpMaxPanels * kPlanWords));
    }
    CK(cudaGetLastError());
    g.init = true;
    return F2_OK;
}

extern uint64_t g_ws_gen;
int ensure_workspace(size_t m, size_t nq, size_t npanels, size_t scratch_words) {
    if (m > g.cap_m || nq > g.cap_q || scratch_words > g.cap_scratch) ++g_ws_gen;
    // a failed allocation leaves the buffer null with capacity 0 (never a stale pointer)
    if (m > g.cap_m) {
        cudaFree(g.P);
        cudaFree(g.pmap);
        g.P = g.pmap = nullptr;
        g.cap_m = 0;
        CK(cudaMalloc(&g.P, sizeof(int64_t) * std::max<size_t>(m, 1)));
        CK(cudaMalloc(&g.pmap, sizeof(int64_t) * std::max<size_t>(m, 1)));
        g.cap_m = m;
    }
    if (scratch_words > g.cap_scratch) {
        cudaFree(g.scratch);
        g.scratch = nullptr;
        g.cap_scratch = 0;
        CK(cudaMalloc(&g.scratch, sizeof(uint64_t) * scratch_words));
        g.cap_scratch = scratch_words;
    }
    if (nq > g.cap_q) {
        cudaFree(g.Qp);
        g.Qp = nullptr;
        g.cap_q = 0;
        CK(cudaMalloc(&g.Qp, sizeof(int64_t) * std::max<size_t>(nq, 1)));
        g.cap_q = nq;
    }
    if (npanels > g.h_r_cap) {
        cudaFreeHost(g.h_r);
        g.h_r = nullptr;
        g.h_r_cap = 0;
        CK(cudaMallocHost(&g.h_r, sizeof(int64_t) * npanels));
        g.h_r_cap = npanels;
    }
    return F2_OK;
}

// expanded operands of the tensor-core Schur: A for every row, B for the trailing
// columns plus the next panel's (t1 and t2 of one panel use disjoint regions)
// (streamed upload: aslots expanded A operands, one per streaming panel, and extra_b
// bytes of B regions for the column groups)
int ensure_f4(size_t m, size_t nw, size_t aslots = 1, size_t extra_b = 0) {
    const size_t a = schur_f4_a_bytes(static_cast<int64_t>(m)) * aslots;
    const size_t b = schur_f4_b_bytes(static_cast<int64_t>(nw)) + schur_f4_b_bytes(kMaxPanelBits / 64) + extra_b;
    if (a > g.cap_f4a || b > g.cap_f4b) ++g_ws_gen;
    if (a > g.cap_f4a) {
        cudaFree(g.f4_ax);
        g.f4_ax = nullptr;
        g.cap_f4a = 0;
        CK(cudaMalloc(&g.f4_ax, a));
        g.cap_f4a = a;
    }
    if (b > g.cap_f4b) {
        cudaFree(g.f4_bx);
        g.f4_bx = nullptr;
        g.cap_f4b = 0;
        CK(cudaMalloc(&g.f4_bx, b));
        g.cap_f4b = b;
    }
    if (!g.f4_claim) CK(cudaMalloc(&g.f4_claim, (2 + kUpGroups) * sizeof(unsigned)));
    return F2_OK;
}

size_t stride_for(size_t ncols) {
    size_t w = (ncols + 63) / 64;
    return (w + 15) / 16 * 16;
}

Mat mat_of(const f2_matrix* a) {
    return Mat{a->d, static_cast<int64_t>(a->m), static_cast<int64_t>(a->n), static_cast<int64_t>(a->stride)};
}

int alloc_matrix(size_t m, size_t n, f2_matrix** out) {
    f2_matrix* a = new f2_matrix;
    a->m = m;
    a->n = n;
    a->stride = stride_for(n);
    a->device = g.device;
    size_t bytes = std::max<size_t>(m * a->stride * 8, 8);
    cudaError_t e = cudaMalloc(&a->d, bytes);
    if (e != cudaSuccess) {
        delete a;
        return cuda_fail(e, "cudaMalloc(matrix)");
    }
    e = cudaMemsetAsync(a->d, 0, bytes, g.stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(matrix)");
    *out = a;
    return F2_OK;
}

// ---- stats ------------------------------------------------------------------
struct Timed {
    int fam;
    cudaEvent_t e0, e1;
    double bytes, bitops;
};
std::vector<Timed> g_timed;

struct LaunchTimer {
    int fam;
    double bytes, bitops;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    LaunchTimer(int f, double by, double bo) : fam(f), bytes(by), bitops(bo) {
        ++g.launches;
        if (g.stats) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, g.stream);
        }
    }
    ~LaunchTimer() {
        if (g.stats) {
            cudaEventRecord(e1, g.stream);
            g_timed.push_back({fam, e0, e1, bytes, bitops});
        }
    }
};

void collect_stats() {
    if (g_timed.empty()) return;
    cudaStreamSynchronize(g.stream);
    for (auto& t : g_timed) {
        float ms = 0;
        cudaEventElapsedTime(&ms, t.e0, t.e1);
        auto& f = g.fam[t.fam];
        f.n += 1;
        f.ms += ms;
        f.bytes += t.bytes;
        f.bitops += t.bitops;
        cudaEventDestroy(t.e0);
        cudaEventDestroy(t.e1);
    }
    g_timed.clear();
}

// ---- event timeline (F2_EVTL=1, non-graph runs only): per-panel marks on the GPU clock
struct EvMark {
    const char* name;
    int64_t panel;
    cudaEvent_t e;
};
std::vector<EvMark> g_evm;
bool g_evtl = false;
inline void evmark(cudaStream_t s, const char* name, int64_t pi) {
    if (!g_evtl) return;
    cudaEvent_t e;
    cudaError_t er = cudaEventCreate(&e);
    if (er == cudaSuccess) er = cudaEventRecord(e, s);
    if (er == cudaSuccess && tune.evtl_sync) er = cudaStreamSynchronize(s);
    if (er != cudaSuccess) std::fprintf(stderr, "evmark %s %lld: %s\n", name, static_cast<long long>(pi), cudaGetErrorString(er));
    g_evm.push_back({name, pi, e});
}
void evdump() {
    if (g_evm.empty()) return;
    cudaDeviceSynchronize();
    for (auto& m : g_evm) {
        float ms = 0;
        const cudaError_t er = cudaEventElapsedTime(&ms, g_evm[0].e, m.e);
        if (er != cudaSuccess) std::fprintf(stderr, "evtl: %s\n", cudaGetErrorString(er));
        std::fprintf(stderr, "EVTL %lld %s %.1f\n", static_cast<long long>(m.panel), m.name, 1e3 * ms);
    }
    for (auto& m : g_evm) cudaEventDestroy(m.e);
    g_evm.clear();
}

// ---- Q of pls_recursive -------------------------------------------------------
// pls_recursive_impl's Q bookkeeping (proj/src/pls.cpp:63-103) replayed from the
// pivot columns: leaf rule :71, cut :74-75, merge :96-98.  The recursion's P,
// packed matrix and Q[0..rank) equal the Gaussian ones; only the tail depends on
// the recursion shape, and only through (m, n, cutoff, pivot columns).
void replay_q(size_t m, size_t n, uint64_t cutoff, const int64_t* piv, size_t npiv, uint64_t* q) {
    for (size_t j = 0; j < n; ++j) q[j] = j;
    if (m == 0 || n == 0) return;
    if (n <= 64 || static_cast<uint64_t>(m) * ((n + 7) / 8) <= cutoff) {
        for (size_t t = 0; t < npiv; ++t) q[t] = static_cast<uint64_t>(piv[t]);
        return;
    }
    size_t n0 = ((n / 2 + 63) / 64) * 64;
    if (n0 >= n) n0 = n / 2;
    size_t r0 = 0;
    while (r0 < npiv && static_cast<size_t>(piv[r0]) < n0) ++r0;
    replay_q(m, n0, cutoff, piv, r0, q);
    const size_t r1 = npiv - r0;
    std::vector<int64_t> sub(r1);
    for (size_t t = 0; t < r1; ++t) sub[t] = piv[r0 + t] - static_cast<int64_t>(n0);
    replay_q(m - r0, n - n0, cutoff, sub.data(), r1, q + n0);
    for (size_t i = n0; i < n; ++i) q[i] += n0;
    for (size_t t = 0; t < r1; ++t) q[r0 + t] = q[n0 + t];
}

// ---- the engine -------------------------------------------------------------
struct EngineOut {
    int64_t rank = 0;
    int64_t dl_rows = -1;  // rows [0, dl_rows) already in g.dl_host (streamed download), -1: none
    std::vector<int64_t> P;   // P[0..rank)
    std::vector<int64_t> Qp;  // pivot columns
};

// Speculative D2H of rows [c, c+W) (see Ctx::dl_host) on the download stream.
int enqueue_download(const Mat& A, int64_t c, unsigned W, cudaStream_t s) {
    if (!g.dl_host || c >= A.m) return F2_OK;
    const int64_t rows = std::min<int64_t>(W, A.m - c);
    const int64_t nw = (A.n + 63) / 64;
    CK(cudaEventRecord(g.dl_ev, s));
    CK(cudaStreamWaitEvent(g.dl_stream, g.dl_ev, 0));
    CK(cudaMemcpy2DAsync(g.dl_host + c * g.dl_pitch, g.dl_pitch * 8, A.w + c * A.stride, A.stride * 8, nw * 8, rows,
                         cudaMemcpyDeviceToHost, g.dl_stream));
    return F2_OK;
}

// The Schur update of one panel as a tensor-core job: rows below the panel's pivots
// (rk = {panel_r, panel_kb} on the device), coefficient bits = the panel's L columns,
// B rows = the pivot rows through the raw-column map, columns [cw0, cw1).
F4Job pls_f4_job(const Mat& A, int64_t pw0, int64_t kbits, int64_t cw0, int64_t cw1, const int64_t* rk,
                 const int64_t* brow) {
    F4Job j{};
    j.C = j.A = j.B = A;
    j.cw0 = j.bw0 = cw0;
    j.cw1 = cw1;
    j.aw0 = pw0;
    j.brow = brow;
    j.rk = rk;
    j.rows_end = A.m;
    j.kbits = kbits;
    return j;
}

// The update of the trailing columns by one finished panel, with look-ahead: the
// enqueue sequence shared by the single-GPU engine and the sharded step.  On entry the
// state holds the panel (its kernel ran, or a non-owner imported it); the row gather
// and the snapshot (one launch) come first.  Then, with trailing words [t0, nw):
//  * lookahead: panel p+1's words [t0, nx) are solved (narrow TRSM) and Schur-updated
//    first, then factor_next(side) enqueues panel p+1's kernel on the side stream
//    while the main stream solves and updates [nx, nw).  Early panels (the trailing
//    update dominates) run "split": the narrow solve + Schur move to the side stream
//    too, so the wide Schur starts right after the gather on the SMs the side chain
//    leaves; late panels (the panel kernel is the critical path) keep them in front.
//  * otherwise every trailing word is solved and updated on the main stream.
// pivots_final(stream) is called once the pivot rows are final in every column.
struct PanelStep {
    Mat A;
    Mat Cf;            // the panel's words (L below the pivots); Cf.w == A.w: the panel itself
    int64_t cw0;       // first word of the panel in Cf
    int64_t p, npanels;
    int64_t width;     // panel bits
    int64_t t0, nw;    // trailing words
    bool lookahead;
    int64_t nx;        // look-ahead: panel p+1 occupies words [t0, nx)
    int side_ctas;     // CTAs of the side chain (0: the Tuning rule)
    // streamed upload: the column groups' streams consume the panel too -- the snapshot
    // and the expanded L21 are made even when no trailing word is in [t0, nw), the
    // gather is recorded in plan, and `gathered` is recorded after it
    bool ext = false;
    uint8_t* ax = nullptr;  // expanded L21 (nullptr: g.f4_ax)
    int64_t* plan = nullptr;
    cudaEvent_t gathered = nullptr;
};

// stats of the sharded schedule: Schur launches timed inside the real schedule
struct SchurTimed {
    int64_t p, c0, c1;
    cudaEvent_t e0, e1;
};
std::vector<SchurTimed>* g_schur_timed = nullptr;  // set while f2_dist_step enqueues with stats on

template <class FactorNext, class PivotsFinal>
int enqueue_panel_step(const PanelStep& ps, cudaStream_t s, cudaStream_t sd, FactorNext factor_next,
                       PivotsFinal pivots_final) {
    const Mat& A = ps.A;
    const int64_t m = A.m, nw = ps.nw, t0 = ps.t0;
    const int nleaves = static_cast<int>((ps.width + 63) / 64);
    int64_t* snap = g.snap + (ps.p % kSnapRing) * kSnapWords;
    if (t0 >= nw && !ps.ext) {
        launch_perm(s, A, nw, g.st, g.pmap, g.scratch);
        ++g.launches;
        return pivots_final(s);
    }
    launch_perm(s, A, nw, g.st, g.pmap, g.scratch, snap, nleaves, &ps.Cf, ps.cw0, ps.plan);
    g.launches += 2;
    if (ps.gathered) CK(cudaEventRecord(ps.gathered, s));
    evmark(s, "gather1", ps.p);
    const bool f4 = tune.f4 && g.f4_ax && ps.width >= 256;  // MMPF (W = 64) keeps the table-apply
    uint8_t* const ax = ps.ax ? ps.ax : g.f4_ax;
    F4Job fj = pls_f4_job(A, 0, ps.width, t0, nw, &g.st->panel_r, g.st->brow);
    fj.A = ps.Cf;
    fj.aw0 = ps.cw0;
    if (f4) {  // L21 expanded on aux beside the narrow work (rk: the live state, stable until the fork)
        CK(cudaEventRecord(g.ax_fork, s));
        CK(cudaStreamWaitEvent(g.aux, g.ax_fork, 0));
        launch_schur_f4_expand_a(g.aux, fj, ax, g.nsm);
        evmark(g.aux, "expand_a", ps.p);
        CK(cudaEventRecord(g.ax_join, g.aux));
    }
    if (t0 >= nw) {  // (ext) nothing of the panel's own columns is left to update
        if (f4) CK(cudaStreamWaitEvent(s, g.ax_join, 0));
        return pivots_final(s);
    }
    fj.rk = snap;
    fj.brow = snap + kSnapBrow;
    TableApply ta{};
    ta.C = A;
    ta.c_r1 = m;
    ta.A = ps.Cf;
    ta.aw0 = ps.cw0;
    ta.kw = nleaves;
    ta.kbits = ps.width;
    ta.B = A;
    ta.brow = snap + kSnapBrow;
    ta.rk = snap;
    ta.row_mode = ROWS_AFTER_PANEL;
    ta.st = g.st;
    const int64_t erows = m - std::min<int64_t>(m, (ps.p + 1) * ps.width);  // rows below the pivots at full rank
    const bool late = 100 * (ps.p + 1) >= tune.late_pct * std::max<int64_t>(ps.npanels, 1);
    const int side = ps.side_ctas > 0 ? ps.side_ctas
                                      : (tune.side_ctas_late > 0 && late ? tune.side_ctas_late : tune.side_ctas);
    const int64_t nx = ps.lookahead ? ps.nx : t0;
    const bool split = ps.lookahead && !late && tune.split_early && f4 && nx < nw;
    const bool late_we = tune.wide_early_pct < 0
                             ? late
                             : 100 * (ps.p + 1) >= tune.wide_early_pct * std::max<int64_t>(ps.npanels, 1);
    const bool wide_early = ps.lookahead && !late_we && tune.early_wide_trsm && nx < nw;
    auto schur = [&](cudaStream_t st, int64_t c0, int64_t c1, int region, int grid) -> int {
        if (c1 <= c0) return F2_OK;
        SchurTimed tm{ps.p, c0, c1, nullptr, nullptr};
        if (g_schur_timed) {
            CK(cudaEventCreate(&tm.e0));
            CK(cudaEventCreate(&tm.e1));
            CK(cudaEventRecord(tm.e0, st));
        }
        if (f4) {
            F4Job j = fj;
            j.cw0 = j.bw0 = c0;
            j.cw1 = c1;
            launch_schur_f4(st, j, ax, g.f4_bx + region * schur_f4_b_bytes(kMaxPanelBits / 64), g.f4_claim + region,
                            grid);
        } else {
            TableApply t = ta;
            t.cw0 = t.bw0 = c0;
            t.cw1 = c1;
            launch_table_apply(st, t, grid, erows);
        }
        if (g_schur_timed) {
            CK(cudaEventRecord(tm.e1, st));
            g_schur_timed->push_back(tm);
        }
        return F2_OK;
    };
    int rc;
    if (wide_early) {  // the wide TRSM (disjoint columns) beside the narrow one
        CK(cudaEventRecord(g.tw_fork, s));
        CK(cudaStreamWaitEvent(g.aux, g.tw_fork, 0));
        launch_panel_trsm_snap(g.aux, A, snap, nleaves, nx, nw, 8);
        evmark(g.aux, "trsm_wide", ps.p);
        CK(cudaEventRecord(g.tw_join, g.aux));
    }
    if (split) {
        // side: narrow TRSM, narrow Schur on `side` CTAs, panel p+1's kernel; main: the wide
        // Schur on the other SMs as soon as the wide TRSM and the L21 expansion are done
        CK(cudaEventRecord(g.la_fork, s));
        CK(cudaStreamWaitEvent(sd, g.la_fork, 0));
        launch_panel_trsm_snap(sd, A, snap, nleaves, t0, nx, 1);
        evmark(sd, "trsm_narrow", ps.p);
        CK(cudaEventRecord(g.nt_done, sd));
        CK(cudaStreamWaitEvent(sd, g.ax_join, 0));
        if ((rc = schur(sd, t0, nx, 0, side))) return rc;
        evmark(sd, "schur_narrow", ps.p);
        if (wide_early) CK(cudaStreamWaitEvent(sd, g.tw_join, 0));  // (see the non-split path)
        factor_next(sd, side);
        evmark(sd, "panel_next", ps.p);
        CK(cudaEventRecord(g.la_join, sd));
        if (wide_early) {
            CK(cudaStreamWaitEvent(s, g.tw_join, 0));
        } else {
            launch_panel_trsm_snap(s, A, snap, nleaves, nx, nw, 8);
            evmark(s, "trsm_wide", ps.p);
        }
        CK(cudaStreamWaitEvent(s, g.nt_done, 0));
        if ((rc = pivots_final(s))) return rc;
        CK(cudaStreamWaitEvent(s, g.ax_join, 0));
        if ((rc = schur(s, nx, nw, 1, g.nsm - side))) return rc;
        evmark(s, "schur_wide", ps.p);
        CK(cudaStreamWaitEvent(s, g.la_join, 0));
        return F2_OK;
    }
    if (ps.lookahead) {
        launch_panel_trsm_snap(s, A, snap, nleaves, t0, nx, 1);
        evmark(s, "trsm_narrow", ps.p);
        if (f4) CK(cudaStreamWaitEvent(s, g.ax_join, 0));
        if ((rc = schur(s, t0, nx, 0, g.nsm))) return rc;
        evmark(s, "schur_narrow", ps.p);
        // (F2_TW_JOIN: the next panel's kernel waits for the early wide TRSM.  A divergence
        // once attributed to the two overlapping was a race inside the old column-form pivot
        // search; they touch disjoint columns)
        if (wide_early && tune.tw_join_at_fork) CK(cudaStreamWaitEvent(s, g.tw_join, 0));
        CK(cudaEventRecord(g.la_fork, s));
        CK(cudaStreamWaitEvent(sd, g.la_fork, 0));
        factor_next(sd, side);
        evmark(sd, "panel_next", ps.p);
        CK(cudaEventRecord(g.la_join, sd));
    }
    if (wide_early) {
        CK(cudaStreamWaitEvent(s, g.tw_join, 0));
    } else {
        launch_panel_trsm_snap(s, A, snap, nleaves, nx, nw, 8);
        evmark(s, "trsm_wide", ps.p);
    }
    if ((rc = pivots_final(s))) return rc;
    if (f4) CK(cudaStreamWaitEvent(s, g.ax_join, 0));
    if ((rc = schur(s, nx, nw, 1, f4 || !ps.lookahead ? g.nsm : g.nsm - side))) return rc;
    evmark(s, "schur_wide", ps.p);
    if (ps.lookahead) CK(cudaStreamWaitEvent(s, g.la_join, 0));
    return F2_OK;
}

// Streamed upload plan (host-buffer entry points).  The matrix crosses PCIe in column
// groups at panel boundaries: group 0 = the first up_g0 panels, the rest in equal groups.
// Panels 0 .. ps-2 are "streaming": panel p's own update covers the main region -- the
// groups already joined into the main stream -- and every other group's stream applies
// the panel to its own words once they have landed (row gather from the recorded plan,
// wide TRSM, Schur, from the panel's snapshot and its own expanded L21).  A group joins
// the main stream when the chain reaches it (before the step whose look-ahead factors
// the group's first panel); all of them join before panel ps-1's step.  Needs the
// tensor-core look-ahead engine and n % 64 == 0 (no tail word to mask).
struct UpPlan {
    bool on = false;
    int ps = 0, ng = 0;
    int64_t gb[kUpGroups + 1] = {};
};

UpPlan upload_plan(int64_t m, int64_t n, unsigned W) {
    UpPlan u;
    const int64_t npanels = (n + W - 1) / W;
    if (!tune.stream_upload || !tune.lookahead || !tune.f4 || g.stats || W < 256 || n % 64 || npanels < 16 ||
        m < 2 * static_cast<int64_t>(W))
        return u;
    const int64_t pwords = W / 64, nw = n / 64, g0 = std::min<int64_t>(tune.up_g0, npanels / 2);
    const int64_t per = (npanels - g0 + tune.up_groups - 2) / (tune.up_groups - 1);
    u.on = true;
    u.ps = static_cast<int>(std::min<int64_t>(tune.up_ps, npanels - 2));
    u.gb[1] = g0 * pwords;
    u.ng = 1;
    while (u.ng < tune.up_groups && u.gb[u.ng] < nw) {
        u.gb[u.ng + 1] = std::min(nw, u.gb[u.ng] + per * pwords);
        ++u.ng;
    }
    u.gb[u.ng] = nw;
    return u;
}

// B regions of the column groups' Schur launches, after the narrow and wide ones
size_t upload_b_offset(const UpPlan& u, int i) {
    size_t o = schur_f4_b_bytes(kMaxPanelBits / 64) + schur_f4_b_bytes(u.gb[u.ng]);
    for (int k = 1; k < i; ++k) o += schur_f4_b_bytes(u.gb[k + 1] - u.gb[k]);
    return o;
}

// One right-looking PLS pass, enqueued on `s`.  poll = snapshot r after every panel
// and stop enqueueing once every row is a pivot (not usable inside a graph capture).
int enqueue_engine(const Mat& A, unsigned W, cudaStream_t s, bool poll) {
    int rc = F2_OK;
    const int64_t m = A.m, n = A.n;
    const int64_t nw = (n + 63) / 64;
    const int64_t npanels = (n + W - 1) / W;
    CK(cudaMemsetAsync(g.st, 0, sizeof(PlsState), s));
#ifdef F2_TIMELINE
    CK(cudaMemsetAsync(&g.st->tl[0][0], 0xff, sizeof(g.st->tl[0]), s));  // min slots
    CK(cudaMemsetAsync(&g.st->tl[2][0], 0xff, sizeof(g.st->tl[2]), s));
#endif
    launch_pmap_init(s, g.pmap, m);
    const UpPlan upl = g.ul_host ? upload_plan(m, n, W) : UpPlan{};
    if (g.ul_host && !upl.on) return fail(F2_INVALID_ARGUMENT, "streamed upload requested outside its plan");
    if (upl.on) {  // column groups on the upload stream; group 0 gates panel 0
        CK(cudaEventRecord(g.up_fork, s));
        CK(cudaStreamWaitEvent(g.up, g.up_fork, 0));
        for (int i = 0; i < upl.ng; ++i) {
            const int64_t w0 = upl.gb[i], w1 = upl.gb[i + 1];
            CK(cudaMemcpy2DAsync(A.w + w0, A.stride * 8, g.ul_host + w0, g.ul_pitch * 8, (w1 - w0) * 8, m,
                                 cudaMemcpyHostToDevice, g.up));
            CK(cudaEventRecord(g.up_ev[i], g.up));
            evmark(g.up, "uploaded", i);
        }
        CK(cudaStreamWaitEvent(s, g.up_ev[0], 0));
        for (int i = 1; i < upl.ng; ++i) CK(cudaStreamWaitEvent(g.grp[i], g.up_ev[i], 0));
    }
    int joined = upl.on ? 1 : 0;  // groups [0, joined) form the main region
    std::vector<cudaEvent_t> evs;
    int64_t checked = 0;
    bool stop = false;

    const bool la = tune.lookahead && !g.stats && npanels > 1;
    // the side kernel is launched cooperatively too: the scheduler then places all its
    // CTAs next to the running Schur update at once (plain launches waited for it to drain)
    auto panel_kernel = [&](cudaStream_t st_, int64_t pi_, int ctas) {
        const int64_t c_ = pi_ * W, cw_ = std::min<int64_t>(W, n - c_);
        const int64_t pw0_ = c_ / 64, pw1_ = pw0_ + (cw_ + 63) / 64;
        launch_panel_pipe(st_, A, pw0_, static_cast<int>(cw_), pw1_, g.st, g.P, g.Qp, g.pmap, 0, g.bar, ctas, true);
    };
    evmark(s, "start", -1);
    if (la) panel_kernel(s, 0, g.nsm);
    evmark(s, "panel0", -1);

    for (int64_t pi = 0; pi < npanels && !stop; ++pi) {
        const int64_t c = pi * W;
        const int64_t cw = std::min<int64_t>(W, n - c);
        const int nleaves = static_cast<int>((cw + 63) / 64);
        const int64_t pw0 = c / 64, pw1 = pw0 + nleaves;
        if (la) {
            // panel pi's kernel ran ahead (panel 0: above; others: on the side stream)
        } else {
            LaunchTimer t(1, 0, 0);
            launch_panel_pipe(s, A, pw0, static_cast<int>(cw), pw1, g.st, g.P, g.Qp, g.pmap, 0, g.bar, g.nsm);
        }
        evmark(s, "gather0", pi);
        if (upl.on && joined < upl.ng) {
            // join the groups the chain has reached: panel pi+1 (factored during this step)
            // must lie in the main region; past the streaming panels, every group
            const int64_t nxw = pi + 1 < npanels && pi < upl.ps - 1 ? (pi + 1) * (W / 64) : nw;
            while (joined < upl.ng && upl.gb[joined] <= nxw) {
                CK(cudaEventRecord(g.grp_ev[joined], g.grp[joined]));
                CK(cudaStreamWaitEvent(s, g.grp_ev[joined], 0));
                evmark(s, "joined", joined);
                ++joined;
            }
            if (joined == upl.ng)  // the streaming panels' rows are final in every column now
                for (int64_t k = 0; k < pi; ++k)
                    if ((rc = enqueue_download(A, k * W, W, s))) return rc;
        }
        if (upl.on && joined < upl.ng) {
            // streaming panel: its own update covers the main region [0, E); the other
            // groups' streams take the rest from the snapshot, L21 in slot pi and the plan
            const int64_t E = upl.gb[joined];
            PanelStep ps{A, A, pw0, pi, npanels, cw, pw1, E, pw1 < E, std::min<int64_t>(E, pw1 + W / 64), 0};
            ps.ext = true;
            ps.ax = g.f4_ax + static_cast<size_t>(pi) * schur_f4_a_bytes(m);
            ps.plan = g.plans + pi * kPlanWords;
            ps.gathered = g.gathered;
            ps.side_ctas = tune.up_side;
            auto factor_next = [&](cudaStream_t sd, int ctas) { panel_kernel(sd, pi + 1, ctas); };
            if ((rc = enqueue_panel_step(ps, s, g.side, factor_next, [](cudaStream_t) { return F2_OK; }))) return rc;
            const int64_t* snap = g.snap + (pi % kSnapRing) * kSnapWords;
            for (int i = joined; i < upl.ng; ++i) {
                cudaStream_t gs = g.grp[i];
                const int64_t w0 = upl.gb[i], w1 = upl.gb[i + 1];
                CK(cudaStreamWaitEvent(gs, g.gathered, 0));
                CK(cudaStreamWaitEvent(gs, g.ax_join, 0));
                launch_plan_perm(gs, A, w0, w1, ps.plan, g.scratch);
                launch_panel_trsm_snap(gs, A, snap, nleaves, w0, w1, 8);
                const F4Job j = pls_f4_job(A, pw0, cw, w0, w1, snap, snap + kSnapBrow);
                launch_schur_f4(gs, j, ps.ax, g.f4_bx + upload_b_offset(upl, i), g.f4_claim + 2 + i, g.nsm);
                g.launches += 5;
                evmark(gs, i == upl.ng - 1 ? "group_last" : "group", pi);
            }
        } else if (la) {
            PanelStep ps{A, A, pw0, pi, npanels, cw, pw1, nw, pw1 < nw, std::min<int64_t>(nw, pw1 + W / 64), 0};
            auto factor_next = [&](cudaStream_t sd, int ctas) { panel_kernel(sd, pi + 1, ctas); };
            auto pivots_final = [&](cudaStream_t st_) { return enqueue_download(A, c, W, st_); };
            if ((rc = enqueue_panel_step(ps, s, g.side, factor_next, pivots_final))) return rc;
        } else {
            {
                LaunchTimer t(3, 0, 0);
                launch_perm(s, A, nw, g.st, g.pmap, g.scratch);
                ++g.launches;  // save + put
            }
            if (pw1 < nw) {
                {
                    LaunchTimer t(2, 0, 0);
                    launch_panel_trsm(s, A, A, pw0, nleaves, pw1, nw, g.st);
                }
                if ((rc = enqueue_download(A, c, W, s))) return rc;
                // work is data dependent; filled in from the pivots after the call
                LaunchTimer t(0, static_cast<double>(pi), -1.0);
                if (tune.f4 && g.f4_ax && cw >= 256 && cw <= 1024) {  // panel_r, panel_kb are adjacent
                    const F4Job fj = pls_f4_job(A, pw0, cw, pw1, nw, &g.st->panel_r, g.st->brow);
                    launch_schur_f4_expand_a(s, fj, g.f4_ax, g.nsm);
                    launch_schur_f4(s, fj, g.f4_ax, g.f4_bx, g.f4_claim, g.nsm);
                } else {
                    TableApply ta{};
                    ta.C = A;
                    ta.c_r1 = m;
                    ta.cw0 = pw1;
                    ta.cw1 = nw;
                    ta.A = A;
                    ta.aw0 = pw0;
                    ta.kw = nleaves;
                    ta.kbits = cw;
                    ta.B = A;
                    ta.bw0 = pw1;
                    ta.brow = g.st->brow;
                    ta.row_mode = ROWS_AFTER_PANEL;
                    ta.st = g.st;
                    launch_table_apply(s, ta, g.nsm, m - std::min<int64_t>(m, c + cw));
                }
            } else if ((rc = enqueue_download(A, c, W, s))) {
                return rc;  // last panel: final after the gather
            }
        }
        if (poll) {  // early exit once every row is a pivot: snapshot r without blocking
            CK(cudaMemcpyAsync(g.h_r + pi, &g.st->r, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, s));
            evs.push_back(ev);
            while (checked < static_cast<int64_t>(evs.size()) && cudaEventQuery(evs[checked]) == cudaSuccess) {
                if (g.h_r[checked] >= m && !(upl.on && joined < upl.ng)) stop = true;
                ++checked;
            }
        }
    }
    if (g.dl_host) {  // join the download stream back into s
        CK(cudaEventRecord(g.dl_join, g.dl_stream));
        CK(cudaStreamWaitEvent(s, g.dl_join, 0));
    }
    CK(cudaGetLastError());
    if (poll) {
        CK(cudaStreamSynchronize(s));
        for (auto ev : evs) cudaEventDestroy(ev);
    }
    return F2_OK;
}

// Graph cache: the launch sequence depends only on (matrix, m, n, stride, W) and the
// workspace buffers, so square-ish factorisations replay one captured CUDA graph
// (per-launch overhead of ~3300 small launches at 64K^2 drops to graph-node cost).
// A few graphs are kept (round-robin eviction): a caller alternating between matrix
// buffers, or between shapes, pays the capture + instantiation (~19 ms at 64K^2) once per
// buffer instead of on every call.
struct GraphCache {
    uint64_t* w = nullptr;
    uint64_t* dl_host = nullptr;
    size_t dl_pitch = 0;
    const uint64_t* ul_host = nullptr;
    size_t ul_pitch = 0;
    int64_t m = 0, n = 0, stride = 0;
    unsigned W = 0;
    uint64_t gen = 0;
    uint64_t launches = 0, kernels = 0;  // enqueued launches / kernel nodes per replay
    cudaGraphExec_t exec = nullptr;
};
constexpr int kGraphSlots = 4;
GraphCache g_graphs[kGraphSlots];
int g_graph_next = 0;
uint64_t g_ws_gen = 1;  // bumped whenever a workspace buffer is reallocated

int run_engine(const Mat& A, unsigned W, EngineOut& out) {
    const int64_t m = A.m, n = A.n;
    out.rank = 0;
    out.P.clear();
    out.Qp.clear();
    if (m == 0 || n == 0) return F2_OK;
    const int64_t nw = (n + 63) / 64;
    const int64_t npanels = (n + W - 1) / W;
    int rc = ensure_workspace(static_cast<size_t>(m), static_cast<size_t>(std::min(m, n)), static_cast<size_t>(npanels),
                              static_cast<size_t>(kMaxMoved) * static_cast<size_t>(A.stride));
    if (rc) return rc;
    const UpPlan upl = g.ul_host ? upload_plan(m, A.n, W) : UpPlan{};
    if (g.ul_host) g.ul_used = true;
    if (tune.f4 && (rc = ensure_f4(static_cast<size_t>(m), static_cast<size_t>(nw), upl.on ? upl.ps : 1,
                                   upl.on ? upload_b_offset(upl, upl.ng) - upload_b_offset(upl, 1) : 0)))
        return rc;
    cudaStream_t s = g.stream;
    const bool use_graph = !g.stats && nw >= 32 && n <= 2 * m && tune.graph;
    g_evtl = !use_graph && tune.evtl;
    if (use_graph) {
        GraphCache* gc = nullptr;
        for (auto& c : g_graphs)
            if (c.exec && c.w == A.w && c.m == m && c.n == n && c.stride == A.stride && c.W == W && c.gen == g_ws_gen &&
                c.dl_host == g.dl_host && c.dl_pitch == g.dl_pitch && c.ul_host == g.ul_host && c.ul_pitch == g.ul_pitch)
                gc = &c;
        if (!gc) {
            gc = &g_graphs[g_graph_next];
            g_graph_next = (g_graph_next + 1) % kGraphSlots;
            // the evicted graph has this one's topology when only the matrix buffer differs:
            // then its executable is updated in place (cheaper than a new instantiation)
            const bool same_shape = gc->exec && gc->m == m && gc->n == n && gc->stride == A.stride && gc->W == W &&
                                    gc->gen == g_ws_gen && gc->dl_host == g.dl_host && gc->dl_pitch == g.dl_pitch &&
                                    gc->ul_host == g.ul_host && gc->ul_pitch == g.ul_pitch;
            if (gc->exec && !same_shape) {
                cudaGraphExecDestroy(gc->exec);
                gc->exec = nullptr;
            }
            cudaGraph_t graph;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            const uint64_t l0 = g.launches;
            rc = enqueue_engine(A, W, s, false);
            const uint64_t per_call = g.launches - l0;
            cudaError_t e = cudaStreamEndCapture(s, &graph);
            if (rc) return rc;
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
            uint64_t nk = 0;
            {  // kernel launches per call = the graph's kernel nodes
                size_t nn = 0;
                cudaGraphGetNodes(graph, nullptr, &nn);
                std::vector<cudaGraphNode_t> nodes(nn);
                if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
                for (auto nd : nodes) {
                    cudaGraphNodeType ty;
                    if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++nk;
                }
            }
            e = cudaErrorUnknown;
            if (gc->exec) {
                cudaGraphExecUpdateResultInfo info;
                e = cudaGraphExecUpdate(gc->exec, graph, &info);
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    cudaGraphExecDestroy(gc->exec);
                    gc->exec = nullptr;
                }
            }
            if (e != cudaSuccess) e = cudaGraphInstantiate(&gc->exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) {
                gc->exec = nullptr;
                return cuda_fail(e, "cudaGraphInstantiate");
            }
            gc->w = A.w;
            gc->dl_host = g.dl_host;
            gc->dl_pitch = g.dl_pitch;
            gc->ul_host = g.ul_host;
            gc->ul_pitch = g.ul_pitch;
            gc->m = m;
            gc->n = n;
            gc->stride = A.stride;
            gc->W = W;
            gc->gen = g_ws_gen;
            gc->launches = per_call;
            gc->kernels = nk;
        } else {
            g.launches += gc->launches;
        }
        g.graph_launches = gc->launches;
        g.graph_kernels = g.last_kernels = gc->kernels;
        CK(cudaGraphLaunch(gc->exec, s));
    } else {
        rc = enqueue_engine(A, W, s, true);
        if (rc) return rc;
    }
    CK(cudaGetLastError());
    evdump();
    int64_t r = 0;
    CK(cudaMemcpyAsync(&r, &g.st->r, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out.rank = r;
    out.P.resize(r);
    out.Qp.resize(r);
    if (r) {
        CK(cudaMemcpy(out.P.data(), g.P, sizeof(int64_t) * r, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(out.Qp.data(), g.Qp, sizeof(int64_t) * r, cudaMemcpyDeviceToHost));
    }
    bool ident = true;
    for (int64_t t = 0; t < r && ident; ++t) ident = out.Qp[t] == t;
    if (!ident) {
        LaunchTimer t(3, 0, 0);
        launch_compress(s, A, r, g.Qp, g.nsm);
    }
    if (g.dl_host) {
        // the speculative copies of panels 0..p are valid while every panel found W pivots
        out.dl_rows = 0;
        if (ident) {
            int64_t t = 0;
            for (int64_t pi = 0; pi < npanels; ++pi) {
                const int64_t c = pi * W, hi = std::min<int64_t>(c + W, m);
                if (c >= m) break;
                int64_t kb = 0;
                while (t < r && out.Qp[t] < c + W) {
                    ++kb;
                    ++t;
                }
                if (kb != hi - c) break;
                out.dl_rows = hi;
            }
        }
        g.dl_done = out.dl_rows;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    // resolve the data-dependent work of the timed Schur launches
    if (g.stats) {
        for (auto& tm : g_timed) {
            if (tm.fam != 0 || tm.bitops >= 0) continue;
            const int64_t pi = static_cast<int64_t>(tm.bytes);
            const int64_t c = pi * W, cw = std::min<int64_t>(W, n - c);
            int64_t before = 0, in = 0;
            for (int64_t t2 = 0; t2 < r; ++t2) {
                if (out.Qp[t2] < c) ++before;
                else if (out.Qp[t2] < c + cw) ++in;
            }
            const double rows = static_cast<double>(m - before - in);
            const double tcols = static_cast<double>(n - c - cw);
            const double tbytes = 8.0 * static_cast<double>(nw - (c + cw) / 64);
            tm.bitops = in ? 2.0 * rows * in * tcols : 0.0;
            // algorithmic HBM bytes: C read+write, the coefficient words, the B rows
            tm.bytes = in ? rows * (2.0 * tbytes + 8.0 * ((cw + 63) / 64)) + in * tbytes : 0.0;
        }
        collect_stats();
    }
    return F2_OK;
}

bool window_ok(const f2_matrix* a, const f2_window& w) {
    return w.r0 <= w.r1 && w.c0 <= w.c1 && w.r1 <= a->m && w.c1 <= a->n;
}

bool full_window(const f2_matrix* a, const f2_window& w) {
    return w.r0 == 0 && w.c0 == 0 && w.r1 == a->m && w.c1 == a->n;
}

// Run the engine on a window: in place for the whole matrix, otherwise on an
// aligned copy that is written back bit-exactly inside the window bounds.
int pls_on_window(f2_matrix* a, const f2_window& w, unsigned W, EngineOut& out) {
    if (full_window(a, w)) return run_engine(mat_of(a), W, out);
    f2_matrix* tmp = nullptr;
    int rc = alloc_matrix(w.r1 - w.r0, w.c1 - w.c0, &tmp);
    if (rc) return rc;
    Mat t = mat_of(tmp);
    launch_extract(g.stream, mat_of(a), static_cast<int64_t>(w.r0), static_cast<int64_t>(w.c0), t);
    rc = run_engine(t, W, out);
    if (!rc) {
        launch_insert(g.stream, mat_of(a), static_cast<int64_t>(w.r0), static_cast<int64_t>(w.c0), t);
        cudaError_t e = cudaStreamSynchronize(g.stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "window insert");
    }
    cudaFree(tmp->d);
    delete tmp;
    return rc;
}

void fill_pq(const EngineOut& o, uint64_t* p, size_t m, uint64_t* q, size_t n, bool recursive, uint64_t cutoff) {
    for (size_t i = 0; i < m; ++i) p[i] = i;
    for (int64_t t = 0; t < o.rank; ++t) p[t] = static_cast<uint64_t>(o.P[t]);
    if (recursive) {
        replay_q(m, n, cutoff, o.Qp.data(), static_cast<size_t>(o.rank), q);
    } else {
        for (size_t j = 0; j < n; ++j) q[j] = j;
        for (int64_t t = 0; t < o.rank; ++t) q[t] = static_cast<uint64_t>(o.Qp[t]);
    }
}

uint64_t default_cutoff() {
    const uint64_t four_mib = uint64_t{4} << 20;
    uint64_t l2 = 0;
    if (const char* env = std::getenv("F2_L2_BYTES")) {
        char* end = nullptr;
        unsigned long long v = std::strtoull(env, &end, 10);
        if (end && *end == '\0' && v > 0) l2 = v;
    }
#if defined(_SC_LEVEL2_CACHE_SIZE)
    if (l2 == 0) {
        long v = sysconf(_SC_LEVEL2_CACHE_SIZE);
        if (v > 0) l2 = static_cast<uint64_t>(v);
    }
#endif
    if (l2 == 0) return four_mib;
    return std::min(l2, four_mib);
}

}  // namespace

// =============================================================================
extern "C" {

const char* f2_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace f2g {
// for the host-side modules (io.cu): same thread-local message as fail()
int set_error(int code, const std::string& msg) { return fail(code, msg); }
int set_cuda_error(cudaError_t e, const char* what) { return cuda_fail(e, what); }
}  // namespace f2g

extern "C" {

int f2_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int f2_set_device(int device) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (g.init && device != g.device) return fail(F2_INVALID_ARGUMENT, "device already initialised");
    g.device = device;
    return ensure_init();
}

int f2_matrix_create(size_t nrows, size_t ncols, f2_matrix** out) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!out) return fail(F2_INVALID_ARGUMENT, "out is NULL");
    int rc = ensure_init();
    if (rc) return rc;
    rc = alloc_matrix(nrows, ncols, out);
    if (rc) return rc;
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

void f2_matrix_destroy(f2_matrix* a) {
    if (!a) return;
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (a->d && a->owns) cudaFree(a->d);
    delete a;
}

size_t f2_matrix_nrows(const f2_matrix* a) { return a ? a->m : 0; }
size_t f2_matrix_ncols(const f2_matrix* a) { return a ? a->n : 0; }
size_t f2_matrix_stride(const f2_matrix* a) { return a ? a->stride : 0; }
uint64_t* f2_matrix_device_ptr(f2_matrix* a) { return a ? a->d : nullptr; }

int f2_matrix_upload(f2_matrix* a, const uint64_t* host, size_t host_stride_words) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || (!host && a->m)) return fail(F2_INVALID_ARGUMENT, "null argument");
    const size_t nw = (a->n + 63) / 64;
    if (host_stride_words < nw) return fail(F2_INVALID_ARGUMENT, "host stride shorter than a row");
    if (a->m == 0 || nw == 0) return F2_OK;
    CK(cudaMemcpy2DAsync(a->d, a->stride * 8, host, host_stride_words * 8, nw * 8, a->m, cudaMemcpyHostToDevice,
                         g.stream));
    // padding bits of the last word must be zero (bitmat.hpp:3-6)
    if (a->n % 64) {
        // cheap: extract onto itself masks the tail word
        Mat t = mat_of(a);
        launch_extract(g.stream, t, 0, 0, t);
    }
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

int f2_matrix_download(const f2_matrix* a, uint64_t* host, size_t host_stride_words) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || (!host && a->m)) return fail(F2_INVALID_ARGUMENT, "null argument");
    const size_t nw = (a->n + 63) / 64;
    if (host_stride_words < nw) return fail(F2_INVALID_ARGUMENT, "host stride shorter than a row");
    if (a->m == 0 || nw == 0) return F2_OK;
    CK(cudaMemcpy2DAsync(host, host_stride_words * 8, a->d, a->stride * 8, nw * 8, a->m, cudaMemcpyDeviceToHost,
                         g.stream));
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

int f2_matrix_copy(f2_matrix* dst, const f2_matrix* src) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!dst || !src) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (dst->m != src->m || dst->n != src->n) return fail(F2_INVALID_ARGUMENT, "shape mismatch");
    if (src->m) CK(cudaMemcpyAsync(dst->d, src->d, src->m * src->stride * 8, cudaMemcpyDeviceToDevice, g.stream));
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

int f2_matrix_clear(f2_matrix* a) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (a->m) CK(cudaMemsetAsync(a->d, 0, a->m * a->stride * 8, g.stream));
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

int f2_matrix_randomize(f2_matrix* a, double density, uint64_t seed) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!(density >= 0.0 && density <= 1.0))
        return fail(F2_INVALID_ARGUMENT, "randomize: density must be in [0, 1]");
    const uint64_t thr = static_cast<uint64_t>(std::llround(density * 9007199254740992.0));
    LaunchTimer t(3, 0, 0);
    launch_randomize(g.stream, mat_of(a), thr, seed);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

// Config 5's generator (the reference has none): one SplitMix64 stream
// (prng.hpp:11-22) from `seed`; per row, draw next() % ncols and reject repeats until
// the row has `weight` distinct ones.  Sequential by construction (a row's draw count
// depends on its rejections), so it runs on the host and uploads the rows.
int f2_matrix_fixed_weight(f2_matrix* a, size_t weight, uint64_t seed) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (weight > a->n) return fail(F2_INVALID_ARGUMENT, "fixed_weight: weight exceeds the column count");
    if (a->m == 0 || a->n == 0) return F2_OK;
    const size_t nw = (a->n + 63) / 64;
    std::vector<uint64_t> rows(a->m * nw, 0);
    uint64_t st = seed;
    auto next = [&st]() {
        uint64_t z = (st += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    for (size_t i = 0; i < a->m; ++i) {
        uint64_t* row = rows.data() + i * nw;
        for (size_t got = 0; got < weight;) {
            const size_t j = static_cast<size_t>(next() % a->n);
            const uint64_t bit = 1ull << (j % 64);
            if (row[j / 64] & bit) continue;
            row[j / 64] |= bit;
            ++got;
        }
    }
    return f2_matrix_upload(a, rows.data(), nw);
}

int f2_matrix_digest(const f2_matrix* a, uint64_t* out) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || !out) return fail(F2_INVALID_ARGUMENT, "null argument");
    launch_digest(g.stream, mat_of(a), g.d_digest);
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, g.d_digest, sizeof(h), cudaMemcpyDeviceToHost, g.stream));
    CK(cudaStreamSynchronize(g.stream));
    *out = h;
    return F2_OK;
}

void* f2_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, std::max<size_t>(bytes, 8)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void f2_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

uint64_t f2_default_cutoff_bytes(void) { return default_cutoff(); }

unsigned f2_auto_table_bits(size_t dim) {
    if (dim < 2) return 1;
    unsigned lg = 0;
    while ((dim >> (lg + 1)) != 0) ++lg;
    if (lg <= 3) return 1;
    return lg - 2 > 8 ? 8 : lg - 2;
}

int f2_set_panel_bits(unsigned bits) {
    if (bits == 0) bits = 1024;
    if (bits % 64 || bits > 1024)
        return fail(F2_INVALID_ARGUMENT, "panel bits must be a multiple of 64 and <= 1024");
    g.panel_bits = bits;
    return F2_OK;
}

// mmpf_pls (mmpf.cpp:81-121): size check :85-86 before touching P/Q; P/Q
// identity-filled :87-88; empty -> 0 :89; k > 8 rejected after the fill :90.
int f2_mmpf_pls(f2_matrix* a, f2_window w, uint64_t* p, size_t plen, uint64_t* q, size_t qlen, unsigned k,
                uint64_t* rank) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || !rank || (!p && plen) || (!q && qlen)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!window_ok(a, w)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t m = w.r1 - w.r0, n = w.c1 - w.c0;
    if (plen != m || qlen != n) return fail(F2_INVALID_ARGUMENT, "mmpf_pls: permutation size mismatch");
    for (size_t i = 0; i < m; ++i) p[i] = i;
    for (size_t j = 0; j < n; ++j) q[j] = j;
    if (m == 0 || n == 0) {
        *rank = 0;
        return F2_OK;
    }
    if (k > 8) return fail(F2_INVALID_ARGUMENT, "mmpf_pls: k must be in 0..8");
    int rc = ensure_init();
    if (rc) return rc;
    g.launches = 0;
    EngineOut o;
    rc = pls_on_window(a, w, tune.mmpf_bits, o);
    if (rc) return rc;
    fill_pq(o, p, m, q, n, false, 0);
    *rank = static_cast<uint64_t>(o.rank);
    return F2_OK;
}

// pls_recursive (pls.cpp:105-113): validate(cfg) :57-61, size check :110-111.
int f2_pls_recursive(f2_matrix* a, f2_window w, uint64_t* p, size_t plen, uint64_t* q, size_t qlen,
                     const f2_elim_config* cfg, uint64_t* rank) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    f2_elim_config c0{0, 0, 0.15, F2_ALG_PLS};
    const f2_elim_config& cfg_ = cfg ? *cfg : c0;
    if (!a || !rank || (!p && plen) || (!q && qlen)) return fail(F2_INVALID_ARGUMENT, "null argument");
    const uint64_t cutoff = cfg_.cutoff_bytes ? cfg_.cutoff_bytes : default_cutoff();
    if (cutoff == 0) return fail(F2_INVALID_ARGUMENT, "cutoff_bytes must be positive");
    if (!(cfg_.hybrid_threshold >= 0.0 && cfg_.hybrid_threshold <= 1.0))
        return fail(F2_INVALID_ARGUMENT, "hybrid_threshold must be in [0, 1]");
    if (!window_ok(a, w)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t m = w.r1 - w.r0, n = w.c1 - w.c0;
    if (plen != m || qlen != n) return fail(F2_INVALID_ARGUMENT, "pls_recursive: permutation size mismatch");
    for (size_t i = 0; i < m; ++i) p[i] = i;
    for (size_t j = 0; j < n; ++j) q[j] = j;
    if (m == 0 || n == 0) {
        *rank = 0;
        return F2_OK;
    }
    // the reference's first leaf is mmpf_pls(.., cfg.k), which rejects k > 8
    if (cfg_.k > 8) return fail(F2_INVALID_ARGUMENT, "mmpf_pls: k must be in 0..8");
    int rc = ensure_init();
    if (rc) return rc;
    g.launches = 0;
    EngineOut o;
    rc = pls_on_window(a, w, g.panel_bits, o);
    if (rc) return rc;
    fill_pq(o, p, m, q, n, true, cutoff);
    *rank = static_cast<uint64_t>(o.rank);
    return F2_OK;
}

// Host-buffer entry points keep one cached device matrix per shape, so a caller
// that decomposes many host matrices pays for the transfers, not for allocation.
static f2_matrix* g_host_mat = nullptr;

static int pls_host(bool recursive, uint64_t* words, size_t nrows, size_t ncols, size_t stride_words, uint64_t* p,
                    uint64_t* q, const f2_elim_config* cfg, unsigned k, uint64_t* rank) {
    // held from the upload to the last download: concurrent callers share g_host_mat
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    int rc;
    if ((rc = ensure_init())) return rc;
    if (!g_host_mat || g_host_mat->m != nrows || g_host_mat->n != ncols) {
        if (g_host_mat) {
            cudaFree(g_host_mat->d);
            delete g_host_mat;
            g_host_mat = nullptr;
        }
        if ((rc = alloc_matrix(nrows, ncols, &g_host_mat))) return rc;
    }
    f2_matrix* a = g_host_mat;
    // pinned host buffer: finished pivot rows stream back while later panels compute, and
    // (upload_plan) the engine uploads the matrix itself, factoring the first panels while
    // the rest is still in flight
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, words) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        nrows > 0 && ncols > 0;
    cudaGetLastError();
    const unsigned W = recursive ? g.panel_bits : tune.mmpf_bits;
    const bool streamed = pinned && stride_words >= (ncols + 63) / 64 &&
                          upload_plan(static_cast<int64_t>(nrows), static_cast<int64_t>(ncols), W).on;
    rc = streamed ? F2_OK : f2_matrix_upload(a, words, stride_words);
    if (!rc) {
        g.dl_host = pinned ? words : nullptr;
        g.dl_pitch = stride_words;
        g.dl_done = -1;
        g.ul_host = streamed ? words : nullptr;
        g.ul_pitch = stride_words;
        g.ul_used = false;
        f2_window w{0, 0, nrows, ncols};
        rc = recursive ? f2_pls_recursive(a, w, p, nrows, q, ncols, cfg, rank)
                       : f2_mmpf_pls(a, w, p, nrows, q, ncols, k, rank);
        g.dl_host = nullptr;
        g.ul_host = nullptr;
        // (an argument error before the engine: the host matrix stays as it was)
        if (streamed && !g.ul_used) return rc;
    }
    if (!rc) {
        const int64_t done = g.dl_done < 0 ? 0 : g.dl_done;
        if (done < static_cast<int64_t>(nrows)) {  // the rest (non-pivot rows, or every row after a fallback)
            const size_t nw = (ncols + 63) / 64;
            CK(cudaMemcpy2DAsync(words + done * stride_words, stride_words * 8, a->d + done * a->stride, a->stride * 8,
                                 nw * 8, nrows - done, cudaMemcpyDeviceToHost, g.stream));
            CK(cudaStreamSynchronize(g.stream));
        }
    }
    return rc;
}

int f2_mmpf_pls_host(uint64_t* words, size_t nrows, size_t ncols, size_t stride_words, uint64_t* p, uint64_t* q,
                     unsigned k, uint64_t* rank) {
    return pls_host(false, words, nrows, ncols, stride_words, p, q, nullptr, k, rank);
}

int f2_pls_recursive_host(uint64_t* words, size_t nrows, size_t ncols, size_t stride_words, uint64_t* p,
                          uint64_t* q, const f2_elim_config* cfg, uint64_t* rank) {
    return pls_host(true, words, nrows, ncols, stride_words, p, q, cfg, 0, rank);
}

int f2_stats_enable(int enable) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g.stats = enable != 0;
    return F2_OK;
}

int f2_stats_get(int kind, uint64_t* launches, double* ms, double* bytes, double* bitops) {
    if (kind < 0 || kind > 3) return fail(F2_INVALID_ARGUMENT, "kind out of range");
    const auto& f = g.fam[kind];
    if (launches) *launches = f.n;
    if (ms) *ms = f.ms;
    if (bytes) *bytes = f.bytes;
    if (bitops) *bitops = f.bitops;
    return F2_OK;
}

int f2_stats_reset(void) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    for (auto& f : g.fam) f = Ctx::Family{};
    return F2_OK;
}

uint64_t f2_last_launch_count(void) { return g.launches; }
uint64_t f2_last_graph_kernels(void) { return g.last_kernels; }

// device timer on the library's stream (bench.py: CUDA events, not host clocks)
static cudaEvent_t g_t0 = nullptr, g_t1 = nullptr;
int f2_timer_start(void) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    int rc = ensure_init();
    if (rc) return rc;
    if (!g_t0) {
        CK(cudaEventCreate(&g_t0));
        CK(cudaEventCreate(&g_t1));
    }
    CK(cudaEventRecord(g_t0, g.stream));
    return F2_OK;
}
int f2_timer_stop(double* ms) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!g_t0 || !ms) return fail(F2_INVALID_ARGUMENT, "timer not started");
    CK(cudaEventRecord(g_t1, g.stream));
    CK(cudaEventSynchronize(g_t1));
    float f = 0;
    CK(cudaEventElapsedTime(&f, g_t0, g_t1));
    *ms = f;
    return F2_OK;
}

// phase clocks recorded by builds compiled with -DF2_LEAF_PROFILE (development aid)
int f2_debug_timeline(unsigned long long* out, int n) {
    if (!g.init || !out || n <= 0) return F2_INVALID_ARGUMENT;
    static unsigned long long tmp[4 * 128];
    CK(cudaMemcpy(tmp, &g.st->tl[0][0], sizeof(tmp), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n && i < 4 * 128; ++i) out[i] = tmp[i];
    return F2_OK;
}

int f2_debug_prof(long long* out, int n) {
    if (!g.init || !out || n <= 0) return F2_INVALID_ARGUMENT;
    long long tmp[64];
    CK(cudaMemcpy(tmp, &g.st->prof[0], sizeof(tmp), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n && i < 64; ++i) out[i] = tmp[i];
    return F2_OK;
}

int f2_debug_clocks(long long* out, int n) {
    if (!g.init || !out || n <= 0) return F2_INVALID_ARGUMENT;
    long long tmp[96];  // dbg[32] then prof[64] (contiguous in PlsState)
    static_assert(offsetof(PlsState, prof) == offsetof(PlsState, dbg) + 32 * sizeof(long long), "dbg/prof layout");
    CK(cudaMemcpy(tmp, &g.st->dbg[0], sizeof(tmp), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n && i < 96; ++i) out[i] = tmp[i];
    return F2_OK;
}

}  // extern "C"

// ---- multiply / triangular solve / permutations ------------------------------
namespace {

bool overlaps(const f2_matrix* x, const f2_window& a, const f2_matrix* y, const f2_window& b) {
    if (x != y) return false;
    const bool rows = a.r0 < b.r1 && b.r0 < a.r1;
    const bool cols = a.c0 < b.c1 && b.c0 < a.c1;
    return rows && cols && a.r0 < a.r1 && b.r0 < b.r1 && a.c0 < a.c1 && b.c0 < b.c1;
}

struct TmpMat {
    f2_matrix* m = nullptr;
    ~TmpMat() {
        if (m) {
            cudaFree(m->d);
            delete m;
        }
    }
};

int extract_tmp(const f2_matrix* a, const f2_window& w, TmpMat& t) {
    int rc = alloc_matrix(w.r1 - w.r0, w.c1 - w.c0, &t.m);
    if (rc) return rc;
    launch_extract(g.stream, mat_of(a), static_cast<int64_t>(w.r0), static_cast<int64_t>(w.c0), mat_of(t.m));
    return F2_OK;
}

// C(p x q) ^= A(p x s) * B(s x q); A and B aligned at (0,0), C at (cr0, word cw0)
void table_mul(const Mat& C, int64_t cr0, int64_t cw0, const Mat& A, int64_t ar0, int64_t aw0, int64_t s,
               const Mat& B, int64_t br0, int64_t bw0, int64_t p, int64_t q) {
    TableApply ta{};
    ta.C = C;
    ta.c_r0 = cr0;
    ta.c_r1 = cr0 + p;
    ta.cw0 = cw0;
    ta.cw1 = cw0 + (q + 63) / 64;
    ta.A = A;
    ta.a_r0 = ar0;
    ta.aw0 = aw0;
    ta.kw = static_cast<int>((s + 63) / 64);
    ta.kbits = s;
    ta.B = B;
    ta.b_r0 = br0;
    ta.bw0 = bw0;
    ta.brow = nullptr;
    ta.row_mode = ROWS_STATIC;
    ta.st = nullptr;
    // algorithmic HBM bytes: C read + written, the coefficient words of every row, the B rows
    const double cbytes = 8.0 * static_cast<double>((q + 63) / 64);
    const double abytes = 8.0 * static_cast<double>((s + 63) / 64);
    LaunchTimer t(0, static_cast<double>(p) * (2.0 * cbytes + abytes) + static_cast<double>(s) * cbytes,
                  2.0 * static_cast<double>(p) * static_cast<double>(s) * static_cast<double>(q));
    // tensor cores once the product is deep and wide enough to fill 128 x 256 x 1024 tiles
    // (F2_SCHUR_M4RM=1 keeps the SMEM table kernel); K is cut into chunks of <= 1024
    if (tune.f4 && s >= 256 && p >= 128 && q >= 256 && ensure_f4(static_cast<size_t>(p), static_cast<size_t>(ta.cw1 - cw0)) == F2_OK) {
        for (int64_t k0 = 0; k0 < s; k0 += kF4MaxK) {
            F4Job j{};
            j.C = C;
            j.c_r0 = cr0;
            j.cw0 = cw0;
            j.cw1 = ta.cw1;
            j.A = A;
            j.a_r0 = ar0;
            j.aw0 = aw0 + k0 / 64;
            j.B = B;
            j.b_r0 = br0 + k0;
            j.bw0 = bw0;
            j.rows_end = p;
            j.kbits = std::min<int64_t>(kF4MaxK, s - k0);
            launch_schur_f4_expand_a(g.stream, j, g.f4_ax, g.nsm);
            launch_schur_f4(g.stream, j, g.f4_ax, g.f4_bx, g.f4_claim, g.nsm);
            g.launches += 3;
        }
        return;
    }
    launch_table_apply(g.stream, ta, g.nsm, p);
}

// B <- L^{-1} B for L = Lm rows/cols [o, o+r) (o % 64 == 0) and B = Bm rows [o, o+r)
void trsm_rec(const Mat& Lm, const Mat& Bm, int64_t o, int64_t r) {
    if (r <= 1) return;
    const int64_t nwb = (Bm.n + 63) / 64;
    if (r <= 1024) {
        Mat lsub{Lm.w + o * Lm.stride + o / 64, r, r, Lm.stride};
        LaunchTimer t(2, 0, 0);
        launch_pivot_trsm(g.stream, Bm, 0, static_cast<int>((r + 63) / 64), 0, nwb, nullptr, PivotSet{2, o, r}, &lsub);
        return;
    }
    int64_t h = (r / 2 + 63) / 64 * 64;
    if (h >= r) h = r / 2;
    trsm_rec(Lm, Bm, o, h);
    // B1 ^= L10 * B0
    table_mul(Bm, o + h, 0, Lm, o + h, o / 64, h, Bm, o, 0, r - h, Bm.n);
    trsm_rec(Lm, Bm, o + h, r - h);
}

}  // namespace

extern "C" {

int f2_addmul(f2_matrix* c, f2_window wc, f2_matrix* a, f2_window wa, f2_matrix* b, f2_window wb, unsigned k) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    (void)k;  // table width is an implementation choice; the product is exact for any k
    if (!a || !b || !c) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!window_ok(a, wa) || !window_ok(b, wb) || !window_ok(c, wc))
        return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t p = wa.r1 - wa.r0, s = wa.c1 - wa.c0, q = wb.c1 - wb.c0;
    if (p != wc.r1 - wc.r0 || s != wb.r1 - wb.r0 || q != wc.c1 - wc.c0)
        return fail(F2_INVALID_ARGUMENT, "addmul: dimension mismatch");
    if (overlaps(c, wc, a, wa) || overlaps(c, wc, b, wb)) return fail(F2_INVALID_ARGUMENT, "addmul: C aliases an input");
    if (p == 0 || s == 0 || q == 0) return F2_OK;
    int rc = ensure_init();
    if (rc) return rc;
    g.launches = 0;
    TmpMat at, bt;
    if ((rc = extract_tmp(a, wa, at)) || (rc = extract_tmp(b, wb, bt))) return rc;
    if (wc.c0 % 64 == 0) {
        table_mul(mat_of(c), static_cast<int64_t>(wc.r0), static_cast<int64_t>(wc.c0 / 64), mat_of(at.m), 0, 0,
                  static_cast<int64_t>(s), mat_of(bt.m), 0, 0, static_cast<int64_t>(p), static_cast<int64_t>(q));
    } else {
        TmpMat ct;
        if ((rc = extract_tmp(c, wc, ct))) return rc;
        table_mul(mat_of(ct.m), 0, 0, mat_of(at.m), 0, 0, static_cast<int64_t>(s), mat_of(bt.m), 0, 0,
                  static_cast<int64_t>(p), static_cast<int64_t>(q));
        launch_insert(g.stream, mat_of(c), static_cast<int64_t>(wc.r0), static_cast<int64_t>(wc.c0), mat_of(ct.m));
        CK(cudaStreamSynchronize(g.stream));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    if (g.stats) collect_stats();
    return F2_OK;
}

int f2_mul_m4rm(const f2_matrix* a, const f2_matrix* b, unsigned k, f2_matrix** out) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || !b || !out) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (a->n != b->m) return fail(F2_INVALID_ARGUMENT, "mul_m4rm: dimension mismatch");
    if (k > 8) return fail(F2_INVALID_ARGUMENT, "mul_m4rm: k must be in 0..8");
    int rc = ensure_init();
    if (rc) return rc;
    g.launches = 0;
    if ((rc = alloc_matrix(a->m, b->n, out))) return rc;
    if (a->m && b->n && a->n)
        table_mul(mat_of(*out), 0, 0, mat_of(a), 0, 0, static_cast<int64_t>(a->n), mat_of(b), 0, 0,
                  static_cast<int64_t>(a->m), static_cast<int64_t>(b->n));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    if (g.stats) collect_stats();
    return F2_OK;
}

int f2_trsm_lower_left_unit(f2_matrix* l, f2_window wl, f2_matrix* b, f2_window wb) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!l || !b) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!window_ok(l, wl) || !window_ok(b, wb)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t r = wl.r1 - wl.r0;
    if (r != wl.c1 - wl.c0) return fail(F2_INVALID_ARGUMENT, "trsm: L must be square");
    if (r != wb.r1 - wb.r0) return fail(F2_INVALID_ARGUMENT, "trsm: dimension mismatch");
    if (r <= 1 || wb.c1 == wb.c0) return F2_OK;
    int rc = ensure_init();
    if (rc) return rc;
    g.launches = 0;
    TmpMat lt, bt;
    if ((rc = extract_tmp(l, wl, lt)) || (rc = extract_tmp(b, wb, bt))) return rc;
    trsm_rec(mat_of(lt.m), mat_of(bt.m), 0, static_cast<int64_t>(r));
    launch_insert(g.stream, mat_of(b), static_cast<int64_t>(wb.r0), static_cast<int64_t>(wb.c0), mat_of(bt.m));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    if (g.stats) collect_stats();
    return F2_OK;
}

// void trsm_upper_left_unit(MatrixWindow u, MatrixWindow b) — mul.hpp:28, mul.cpp:133-155:
// B <- U^{-1} B, U unit upper triangular (its lower part ignored).  With R the row/column
// reversal, U^{-1} B = R (R U R)^{-1} R B: the lower solver on reversed copies.
int f2_trsm_upper_left_unit(f2_matrix* u, f2_window wu, f2_matrix* b, f2_window wb) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!u || !b) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!window_ok(u, wu) || !window_ok(b, wb)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t r = wu.r1 - wu.r0;
    if (r != wu.c1 - wu.c0) return fail(F2_INVALID_ARGUMENT, "trsm: U must be square");
    if (r != wb.r1 - wb.r0) return fail(F2_INVALID_ARGUMENT, "trsm: dimension mismatch");
    if (r <= 1 || wb.c1 == wb.c0) return F2_OK;
    int rc = ensure_init();
    if (rc) return rc;
    g.launches = 0;
    TmpMat ut, bt, lrev, brev;
    if ((rc = extract_tmp(u, wu, ut)) || (rc = extract_tmp(b, wb, bt))) return rc;
    if ((rc = alloc_matrix(r, r, &lrev.m)) || (rc = alloc_matrix(r, wb.c1 - wb.c0, &brev.m))) return rc;
    const int64_t rr = static_cast<int64_t>(r);
    launch_reverse_square(g.stream, mat_of(lrev.m), mat_of(ut.m), rr);
    std::vector<int64_t> rev(r);
    for (int64_t i = 0; i < rr; ++i) rev[i] = rr - 1 - i;
    int64_t* dmap = nullptr;
    CK(cudaMalloc(&dmap, sizeof(int64_t) * r));
    CK(cudaMemcpyAsync(dmap, rev.data(), sizeof(int64_t) * r, cudaMemcpyHostToDevice, g.stream));
    const int64_t nwb = static_cast<int64_t>(bt.m->stride);
    launch_gather_rows(g.stream, mat_of(brev.m), mat_of(bt.m), dmap, rr, nwb);
    trsm_rec(mat_of(lrev.m), mat_of(brev.m), 0, rr);
    launch_gather_rows(g.stream, mat_of(bt.m), mat_of(brev.m), dmap, rr, nwb);
    launch_insert(g.stream, mat_of(b), static_cast<int64_t>(wb.r0), static_cast<int64_t>(wb.c0), mat_of(bt.m));
    const cudaError_t e = cudaStreamSynchronize(g.stream);
    cudaFree(dmap);
    if (e != cudaSuccess) return cuda_fail(e, "trsm_upper_left_unit");
    if (g.stats) collect_stats();
    return F2_OK;
}

int f2_compress_columns(f2_matrix* a, uint64_t rank, const uint64_t* q, size_t qlen) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || (!q && qlen)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (rank > a->m || rank > qlen) return fail(F2_INVALID_ARGUMENT, "compress_columns: rank out of range");
    for (uint64_t j = 0; j < rank; ++j)
        if (q[j] >= a->n || j >= a->n) return fail(F2_INVALID_ARGUMENT, "compress_columns: column out of range");
    if (rank == 0) return F2_OK;
    if (a->stride * 8 > 200 * 1024) return fail(F2_INVALID_ARGUMENT, "compress_columns: row wider than 1.6M bits");
    int rc = ensure_init();
    if (rc) return rc;
    int64_t* dq = nullptr;
    CK(cudaMalloc(&dq, sizeof(int64_t) * rank));
    std::vector<int64_t> hq(q, q + rank);
    CK(cudaMemcpyAsync(dq, hq.data(), sizeof(int64_t) * rank, cudaMemcpyHostToDevice, g.stream));
    launch_col_swaps(g.stream, mat_of(a), static_cast<int64_t>(rank), dq, g.nsm);
    cudaError_t e = cudaStreamSynchronize(g.stream);
    cudaFree(dq);
    if (e != cudaSuccess) return cuda_fail(e, "compress_columns");
    return F2_OK;
}

int f2_apply_rows(f2_matrix* a, f2_window w, const uint64_t* p, size_t plen, int inverse) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || (!p && plen)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!window_ok(a, w)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t m = w.r1 - w.r0;
    if (plen > m) return fail(F2_INVALID_ARGUMENT, "apply_rows: permutation longer than rows");
    for (size_t i = 0; i < plen; ++i)
        if (p[i] >= m) return fail(F2_INVALID_ARGUMENT, "apply_rows: entry out of range");
    if (m == 0 || w.c1 == w.c0) return F2_OK;
    int rc = ensure_init();
    if (rc) return rc;
    std::vector<int64_t> idx(m);
    for (size_t i = 0; i < m; ++i) idx[i] = static_cast<int64_t>(i);
    if (!inverse) {
        for (size_t i = 0; i < plen; ++i) std::swap(idx[i], idx[p[i]]);
    } else {
        for (size_t i = plen; i-- > 0;) std::swap(idx[i], idx[p[i]]);
    }
    TmpMat t1, t2;
    if ((rc = extract_tmp(a, w, t1))) return rc;
    if ((rc = alloc_matrix(m, w.c1 - w.c0, &t2.m))) return rc;
    int64_t* dmap = nullptr;
    CK(cudaMalloc(&dmap, sizeof(int64_t) * m));
    CK(cudaMemcpyAsync(dmap, idx.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, g.stream));
    launch_gather_rows(g.stream, mat_of(t2.m), mat_of(t1.m), dmap, static_cast<int64_t>(m),
                       static_cast<int64_t>(t1.m->stride));
    launch_insert(g.stream, mat_of(a), static_cast<int64_t>(w.r0), static_cast<int64_t>(w.c0), mat_of(t2.m));
    cudaError_t e = cudaStreamSynchronize(g.stream);
    cudaFree(dmap);
    if (e != cudaSuccess) return cuda_fail(e, "apply_rows");
    return F2_OK;
}

}  // extern "C"

// ---- column-sharded PLS (paper_1006_1744_b200/dist.py) --------------------------------
// Rank k of N holds the panels p = k, k+N, ... (W bits each) side by side in a local
// matrix with all m rows.  P, the pivot columns and every packed column equal the
// single-GPU engine's (same pivot rule, same row operations per column).  Every call
// below only ENQUEUES work on the caller's streams (torch streams in dist.py); nothing
// waits on the GPU before f2_dist_finish, except f2_dist_header_rk, which dist.py calls
// lagged by three panels.
//   f2_dist_factor   owner of panel p: the panel kernel on its columns, then the header
//                    and the panel's words of rows >= panel_r into an exchange buffer,
//                    read through the virtual row order (the buffer can leave before
//                    the owner's own row gather)
//   -- dist.py broadcasts the buffer tail [r_lo * W/64, end) (NCCL over NVLink) --
//   f2_dist_step     every rank, panel p: (non-owner) header -> state, P, Q prefix and
//                    the L11^{-1} maps from the words; row gather over all local columns;
//                    snapshot; panel TRSM + Schur update of the local trailing columns.
//                    Look-ahead when this rank owns panel p+1: its columns first, then
//                    f2_dist_factor(p+1) on the side stream beside the rest, exactly the
//                    single-GPU engine's schedule (enqueue_engine)
//   f2_dist_note     (kb, panel_r) of a buffer's header to pinned memory + an event, on
//                    the stream where the buffer became valid
namespace {
struct DistState {
    int64_t m = 0, ncols = 0;
    unsigned W = 0;
    int64_t npanels = 0;
    int64_t* h_rk = nullptr;  // pinned [npanels][2]: (kb, panel_r)
    size_t cap = 0;
    std::vector<cudaEvent_t> ev;
    std::vector<SchurTimed> timed;  // stats: Schur launches of the timed schedule, work resolved at finish
};
DistState gd;

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void dist_factor_enqueue(const Mat& A, int64_t pw0, unsigned width, int64_t col, uint64_t* buf, int ctas,
                         cudaStream_t s) {
    const int nleaves = static_cast<int>((width + 63) / 64);
    launch_panel_pipe(s, A, pw0, static_cast<int>(width), pw0 + nleaves, g.st, g.P, g.Qp, g.pmap, col - 64 * pw0,
                      g.bar, ctas, true);
    launch_dist_export(s, A, pw0, nleaves, g.st, g.pmap, g.P, buf, static_cast<int>(gd.W), col, g.nsm);
}
}  // namespace

extern "C" {

size_t f2_dist_buffer_words(size_t nrows, unsigned panel_bits) {
    return nrows * (panel_bits / 64) + static_cast<size_t>(dist_header_words(static_cast<int>(panel_bits)));
}

int f2_dist_begin(f2_matrix* a, unsigned panel_bits, size_t npanels, void* stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (panel_bits == 0 || panel_bits % 128 || panel_bits > 1024)
        return fail(F2_INVALID_ARGUMENT, "panel bits must be a multiple of 128 and <= 1024");
    int rc = ensure_init();
    if (rc) return rc;
    const size_t m = std::max<size_t>(a->m, 1);
    if ((rc = ensure_workspace(m, m, npanels + 1, static_cast<size_t>(kMaxMoved) * a->stride))) return rc;
    if (tune.f4 && (rc = ensure_f4(m, (a->n + 63) / 64))) return rc;
    if (npanels > gd.cap) {
        cudaFreeHost(gd.h_rk);
        gd.h_rk = nullptr;
        gd.cap = 0;
        CK(cudaMallocHost(&gd.h_rk, sizeof(int64_t) * 2 * npanels));
        gd.cap = npanels;
    }
    while (gd.ev.size() < npanels) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        gd.ev.push_back(e);
    }
    gd.m = static_cast<int64_t>(a->m);
    gd.ncols = static_cast<int64_t>(a->n);
    gd.W = panel_bits;
    gd.npanels = static_cast<int64_t>(npanels);
    cudaStream_t s = as_stream(stream);
    CK(cudaMemsetAsync(g.st, 0, sizeof(PlsState), s));
    launch_pmap_init(s, g.pmap, static_cast<int64_t>(a->m));
    CK(cudaGetLastError());
    return F2_OK;
}

int f2_dist_factor(f2_matrix* a, size_t pw0, unsigned width_bits, uint64_t panel_col, uint64_t* buf, int ctas,
                   void* stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || !buf) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (width_bits == 0 || width_bits > gd.W || (pw0 * 64 + width_bits) > a->n)
        return fail(F2_INVALID_ARGUMENT, "panel out of range");
    dist_factor_enqueue(mat_of(a), static_cast<int64_t>(pw0), width_bits, static_cast<int64_t>(panel_col), buf,
                        ctas > 0 && ctas <= g.nsm ? ctas : g.nsm, as_stream(stream));
    CK(cudaGetLastError());
    return F2_OK;
}

int f2_dist_step(f2_matrix* a, int64_t p, int owner, size_t pw0, unsigned width_bits, const uint64_t* buf,
                 size_t tw0, int lookahead, unsigned next_width, uint64_t next_col, uint64_t* next_buf, int side_ctas,
                 void* main_stream, void* side_stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || !buf || (lookahead && !next_buf)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (width_bits == 0 || width_bits > gd.W || next_width > gd.W) return fail(F2_INVALID_ARGUMENT, "panel width out of range");
    const Mat A = mat_of(a);
    const int64_t m = A.m, nw = (A.n + 63) / 64, ws = gd.W / 64;
    const int nleaves = static_cast<int>((width_bits + 63) / 64);
    cudaStream_t s = as_stream(main_stream), sd = as_stream(side_stream);
    if (lookahead && static_cast<int64_t>(tw0) >= nw)
        return fail(F2_INVALID_ARGUMENT, "look-ahead without local trailing columns");
    const Mat Bw{const_cast<uint64_t*>(buf), m, static_cast<int64_t>(gd.W), ws};  // the broadcast words
    if (!owner) {
        launch_dist_import(s, g.st, g.pmap, g.P, g.Qp, reinterpret_cast<const int64_t*>(buf + m * ws),
                           static_cast<int>(gd.W));
        launch_panel_lmaps(s, Bw, 0, nleaves, g.st);
    }
    PanelStep ps{A, owner ? A : Bw, owner ? static_cast<int64_t>(pw0) : 0, p, gd.npanels, width_bits,
                 static_cast<int64_t>(tw0), nw, lookahead != 0,
                 std::min<int64_t>(nw, static_cast<int64_t>(tw0) + (next_width + 63) / 64), side_ctas};
    auto factor_next = [&](cudaStream_t st_, int ctas) {
        dist_factor_enqueue(A, static_cast<int64_t>(tw0), next_width, static_cast<int64_t>(next_col), next_buf,
                            std::min(ctas, g.nsm), st_);
    };
    g_schur_timed = g.stats ? &gd.timed : nullptr;  // resolved at f2_dist_finish
    const int rc = enqueue_panel_step(ps, s, sd, factor_next, [](cudaStream_t) { return F2_OK; });
    g_schur_timed = nullptr;
    if (rc) return rc;
    CK(cudaGetLastError());
    return F2_OK;
}

int f2_dist_note(const uint64_t* buf, int64_t p, void* stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!buf || p < 0 || p >= gd.npanels) return fail(F2_INVALID_ARGUMENT, "panel out of range");
    cudaStream_t s = as_stream(stream);
    CK(cudaMemcpyAsync(gd.h_rk + 2 * p, buf + gd.m * (gd.W / 64), 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(gd.ev[p], s));
    return F2_OK;
}

int f2_dist_header_rk(int64_t p, uint64_t* kb, uint64_t* r0) {
    if (p < 0 || p >= gd.npanels || !kb || !r0) return fail(F2_INVALID_ARGUMENT, "panel out of range");
    CK(cudaEventSynchronize(gd.ev[p]));
    *kb = static_cast<uint64_t>(gd.h_rk[2 * p]);
    *r0 = static_cast<uint64_t>(gd.h_rk[2 * p + 1]);
    return F2_OK;
}

// rank, P (LAPACK transpositions, identity past the rank) and the pivot columns; waits
// for `stream` (the caller joins its other streams into it first)
int f2_dist_finish(f2_matrix* a, void* stream, uint64_t* rank, uint64_t* p, size_t plen, uint64_t* pivcols,
                   size_t qcap) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || !rank || (!p && plen) || (!pivcols && qcap)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (plen != a->m) return fail(F2_INVALID_ARGUMENT, "P length must equal the row count");
    cudaStream_t s = as_stream(stream);
    int64_t r = 0;
    CK(cudaMemcpyAsync(&r, &g.st->r, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (static_cast<size_t>(r) > qcap) return fail(F2_INVALID_ARGUMENT, "pivot column buffer too small");
    std::vector<int64_t> tmp(static_cast<size_t>(r));
    for (size_t i = 0; i < plen; ++i) p[i] = i;
    if (r) {
        CK(cudaMemcpy(tmp.data(), g.P, sizeof(int64_t) * r, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < r; ++t) p[t] = static_cast<uint64_t>(tmp[t]);
        CK(cudaMemcpy(tmp.data(), g.Qp, sizeof(int64_t) * r, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < r; ++t) pivcols[t] = static_cast<uint64_t>(tmp[t]);
    }
    *rank = static_cast<uint64_t>(r);
    // stats: each timed Schur launch's work from its panel's header, 2 * rows * kb * columns
    for (auto& tm : gd.timed) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, tm.e0, tm.e1));
        const int64_t kb = gd.h_rk[2 * tm.p], r0 = gd.h_rk[2 * tm.p + 1];
        const double rows = static_cast<double>(gd.m - r0 - kb);
        const double cols = static_cast<double>(std::min<int64_t>(64 * tm.c1, gd.ncols) - 64 * tm.c0);
        auto& f = g.fam[0];
        f.n += 1;
        f.ms += ms;
        f.bitops += 2.0 * rows * static_cast<double>(kb) * cols;
        f.bytes += kb ? rows * 2.0 * 8.0 * static_cast<double>(tm.c1 - tm.c0) : 0.0;
        cudaEventDestroy(tm.e0);
        cudaEventDestroy(tm.e1);
    }
    gd.timed.clear();
    return F2_OK;
}

// A non-owning matrix over caller device memory (e.g. a torch tensor of m x stride
// int64 words; stride a multiple of 16 words): the sharded schedule's local shards
int f2_matrix_view(uint64_t* dev, size_t nrows, size_t ncols, size_t stride_words, f2_matrix** out) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!out || (!dev && nrows)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (stride_words < (ncols + 63) / 64 || stride_words % 16)
        return fail(F2_INVALID_ARGUMENT, "view stride must cover a row and be a multiple of 16 words");
    int rc = ensure_init();
    if (rc) return rc;
    f2_matrix* v = new f2_matrix;
    v->m = nrows;
    v->n = ncols;
    v->stride = stride_words;
    v->d = dev;
    v->device = g.device;
    v->owns = false;
    *out = v;
    return F2_OK;
}

// compress_columns of a packed PLS result given its pivot columns (k_compress)
int f2_pls_compress(f2_matrix* a, uint64_t rank, const uint64_t* pivcols) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || (!pivcols && rank)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (rank == 0) return F2_OK;
    int rc = ensure_init();
    if (rc) return rc;
    if ((rc = ensure_workspace(a->m, rank, 1, static_cast<size_t>(kMaxMoved) * a->stride))) return rc;
    std::vector<int64_t> q(pivcols, pivcols + rank);
    bool ident = true;
    for (uint64_t t = 0; t < rank; ++t) ident &= q[t] == static_cast<int64_t>(t);
    if (ident) return F2_OK;
    CK(cudaMemcpyAsync(g.Qp, q.data(), sizeof(int64_t) * rank, cudaMemcpyHostToDevice, g.stream));
    launch_compress(g.stream, mat_of(a), static_cast<int64_t>(rank), g.Qp, g.nsm);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

// pls_recursive's Q (tail included) from the pivot columns — host only (pls.cpp:63-103)
int f2_recursive_q(size_t m, size_t n, uint64_t cutoff, uint64_t rank, const uint64_t* pivcols, uint64_t* q) {
    if (!q && n) return fail(F2_INVALID_ARGUMENT, "null argument");
    std::vector<int64_t> piv(pivcols, pivcols + rank);
    replay_q(m, n, cutoff ? cutoff : default_cutoff(), piv.data(), static_cast<size_t>(rank), q);
    return F2_OK;
}

}  // extern "C"

// ---- echelonize -------------------------------------------------------------------
namespace {

// RREF of the original matrix from a packed PLS result in the aligned matrix T
// (rref_from_pls, pls.cpp:128-155).  The reduced rows are U^{-1} S, U = S at the
// pivot columns (unit upper triangular): a backward substitution, run as the
// forward solver on row- and column-reversed coefficients.
int rref_on(f2_matrix* t, uint64_t rank, const std::vector<int64_t>& q) {
    const int64_t m = static_cast<int64_t>(t->m);
    const int64_t r = static_cast<int64_t>(rank);
    int rc;
    if ((rc = ensure_workspace(t->m, std::max<size_t>(t->m, rank) + 1, 1, static_cast<size_t>(kMaxMoved) * t->stride)))
        return rc;
    if (r) CK(cudaMemcpyAsync(g.Qp, q.data(), sizeof(int64_t) * r, cudaMemcpyHostToDevice, g.stream));
    launch_rref_prepare(g.stream, mat_of(t), r, g.Qp);
    if (r > 1) {
        TmpMat lrev, xrev;
        if ((rc = alloc_matrix(rank, rank, &lrev.m)) || (rc = alloc_matrix(rank, t->n, &xrev.m))) return rc;
        launch_rref_coeffs(g.stream, mat_of(t), r, g.Qp, mat_of(lrev.m), g.nsm);
        std::vector<int64_t> rev(rank);
        for (int64_t i = 0; i < r; ++i) rev[i] = r - 1 - i;
        int64_t* dmap = nullptr;
        CK(cudaMalloc(&dmap, sizeof(int64_t) * rank));
        CK(cudaMemcpyAsync(dmap, rev.data(), sizeof(int64_t) * rank, cudaMemcpyHostToDevice, g.stream));
        launch_gather_rows(g.stream, mat_of(xrev.m), mat_of(t), dmap, r, static_cast<int64_t>(t->stride));
        trsm_rec(mat_of(lrev.m), mat_of(xrev.m), 0, r);
        launch_gather_rows(g.stream, mat_of(t), mat_of(xrev.m), dmap, r, static_cast<int64_t>(t->stride));
        cudaError_t e = cudaStreamSynchronize(g.stream);
        cudaFree(dmap);
        if (e != cudaSuccess) return cuda_fail(e, "rref");
    }
    (void)m;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

int rref_window(f2_matrix* a, const f2_window& w, uint64_t rank, const std::vector<int64_t>& q) {
    if (full_window(a, w)) return rref_on(a, rank, q);
    TmpMat t;
    int rc = extract_tmp(a, w, t);
    if (rc) return rc;
    if ((rc = rref_on(t.m, rank, q))) return rc;
    launch_insert(g.stream, mat_of(a), static_cast<int64_t>(w.r0), static_cast<int64_t>(w.c0), mat_of(t.m));
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

}  // namespace

extern "C" {

// void rref_from_pls(MatrixWindow a, size_t rank, span<const size_t> q) — pls.cpp:128-155;
// validation as pls.cpp:130-135.
int f2_rref_from_pls(f2_matrix* a, f2_window w, uint64_t rank, const uint64_t* q, size_t qlen) {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!a || (!q && qlen)) return fail(F2_INVALID_ARGUMENT, "null argument");
    if (!window_ok(a, w)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    const size_t m = w.r1 - w.r0, n = w.c1 - w.c0;
    if (rank > m || rank > n || qlen < rank) return fail(F2_INVALID_ARGUMENT, "rref_from_pls: rank out of range");
    for (uint64_t t = 0; t < rank; ++t)
        if (q[t] >= n || q[t] < t || (t > 0 && q[t] <= q[t - 1]))
            return fail(F2_INVALID_ARGUMENT, "rref_from_pls: Q is not a pivot-column prefix");
    if (m == 0 || n == 0) return F2_OK;
    int rc = ensure_init();
    if (rc) return rc;
    std::vector<int64_t> qq(q, q + rank);
    return rref_window(a, w, rank, qq);
}

// Echelonize: reduced row echelon form via PLS + rref_from_pls (the reference's
// rref with Algorithm::pls, acceptance.cpp:39-44 / f2mat rref).  The RREF is
// unique, so this equals gauss_rref / m4ri_rref / hybrid_rref on the same input.
int f2_rref(f2_matrix* a, f2_window w, const f2_elim_config* cfg, uint64_t* rank) {
    if (!a || !rank) return fail(F2_INVALID_ARGUMENT, "null argument");
    {
        std::lock_guard<std::recursive_mutex> lk(g_mu);
        if (!window_ok(a, w)) return fail(F2_OUT_OF_RANGE, "MatrixWindow: invalid bounds");
    }
    const size_t m = w.r1 - w.r0, n = w.c1 - w.c0;
    std::vector<uint64_t> p(m), q(n);
    int rc = f2_pls_recursive(a, w, p.data(), m, q.data(), n, cfg, rank);
    if (rc) return rc;
    return f2_rref_from_pls(a, w, *rank, q.data(), static_cast<size_t>(*rank));
}

// m4ri_rref(BitMatrix&, k, full) — m4ri.hpp:41, m4ri.cpp:68-87.  full: the RREF (unique,
// so PLS + rref_from_pls gives it bit for bit).  !full: M4RI's echelon form, U (the PLS
// pivot rows in original columns) with every block of consecutive pivots that one
// gauss_submatrix call forms (m4ri.cpp:45-67, blocks of <= k0 = k or auto_table_bits
// columns, cut at a pivot-less column) reduced inside the block.
int f2_m4ri_rref(f2_matrix* a, unsigned k, int full, uint64_t* rank) {
    if (!a || !rank) return fail(F2_INVALID_ARGUMENT, "null argument");
    const size_t m = a->m, n = a->n;
    *rank = 0;
    if (m == 0 || n == 0) return F2_OK;
    if (k > 8) return fail(F2_INVALID_ARGUMENT, "m4ri_rref: k must be in 0..8");
    const f2_window w{0, 0, m, n};
    std::vector<uint64_t> p(m), q(n);
    int rc = f2_pls_recursive(a, w, p.data(), m, q.data(), n, nullptr, rank);
    if (rc) return rc;
    if (full) return f2_rref_from_pls(a, w, *rank, q.data(), static_cast<size_t>(*rank));
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    const int64_t r = static_cast<int64_t>(*rank);
    if ((rc = ensure_workspace(m, std::max<size_t>(m, *rank) + 1, 1, static_cast<size_t>(kMaxMoved) * a->stride)))
        return rc;
    std::vector<int64_t> qq(q.begin(), q.begin() + r);
    // the blocks of m4ri_rref's column walk (:73-85) from the pivot columns
    const unsigned k0 = k ? k : f2_auto_table_bits(std::min(m, n));
    std::vector<int64_t> bstart;
    {
        size_t rr = 0, c = 0;
        while (rr < m && c < n) {
            const size_t kc = std::min<size_t>(k0, n - c);
            size_t kbar = 0;
            while (kbar < kc && rr + kbar < static_cast<size_t>(r) && static_cast<size_t>(qq[rr + kbar]) == c + kbar) ++kbar;
            if (kbar) {
                bstart.push_back(static_cast<int64_t>(rr));
                rr += kbar;
                c += kbar;
            }
            if (kbar != kc) ++c;
        }
        bstart.push_back(r);
    }
    if (r) CK(cudaMemcpyAsync(g.Qp, qq.data(), sizeof(int64_t) * r, cudaMemcpyHostToDevice, g.stream));
    launch_rref_prepare(g.stream, mat_of(a), r, g.Qp);  // U in original columns, rows >= rank zero
    const int64_t nb = static_cast<int64_t>(bstart.size()) - 1;
    if (nb > 0) {
        int64_t* dstart = nullptr;
        CK(cudaMalloc(&dstart, sizeof(int64_t) * bstart.size()));
        CK(cudaMemcpyAsync(dstart, bstart.data(), sizeof(int64_t) * bstart.size(), cudaMemcpyHostToDevice, g.stream));
        launch_block_backsub(g.stream, mat_of(a), dstart, g.Qp, nb, g.nsm);
        const cudaError_t e = cudaStreamSynchronize(g.stream);
        cudaFree(dstart);
        if (e != cudaSuccess) return cuda_fail(e, "m4ri echelon");
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g.stream));
    return F2_OK;
}

namespace {
int validate_cfg(const f2_elim_config& c) {  // pls.cpp:57-61
    if ((c.cutoff_bytes ? c.cutoff_bytes : default_cutoff()) == 0)
        return fail(F2_INVALID_ARGUMENT, "cutoff_bytes must be positive");
    if (!(c.hybrid_threshold >= 0.0 && c.hybrid_threshold <= 1.0))
        return fail(F2_INVALID_ARGUMENT, "hybrid_threshold must be in [0, 1]");
    return F2_OK;
}
}  // namespace

// hybrid_rref(BitMatrix&, cfg) — pls.hpp:61, pls.cpp:163-198: its result is the RREF of A
// whatever the density switch decides, so PLS + rref_from_pls gives it bit for bit.
// k > 8 is rejected (the reference's pls_recursive leaf rejects it once the switch fires).
int f2_hybrid_rref(f2_matrix* a, const f2_elim_config* cfg, uint64_t* rank) {
    if (!a || !rank) return fail(F2_INVALID_ARGUMENT, "null argument");
    const f2_elim_config c0{0, 0, 0.15, F2_ALG_HYBRID};
    const f2_elim_config& c = cfg ? *cfg : c0;
    int rc = validate_cfg(c);
    if (rc) return rc;
    *rank = 0;
    if (a->m == 0 || a->n == 0) return F2_OK;
    if (c.k > 8) return fail(F2_INVALID_ARGUMENT, "hybrid_rref: k must be in 0..8");
    return f2_rref(a, f2_window{0, 0, a->m, a->n}, &c, rank);
}

// rank(const BitMatrix&, cfg) — pls.hpp:64, pls.cpp:200-216: rank on a working copy, with
// the validation of the configured algorithm (the rank itself does not depend on it).
int f2_rank(const f2_matrix* a, const f2_elim_config* cfg, uint64_t* rank) {
    if (!a || !rank) return fail(F2_INVALID_ARGUMENT, "null argument");
    const f2_elim_config c0{0, 0, 0.15, F2_ALG_PLS};
    const f2_elim_config& c = cfg ? *cfg : c0;
    if (c.algorithm < F2_ALG_GAUSS || c.algorithm > F2_ALG_HYBRID)
        return fail(F2_INVALID_ARGUMENT, "rank: unknown algorithm");
    if (c.algorithm == F2_ALG_PLS || c.algorithm == F2_ALG_HYBRID) {
        int rc = validate_cfg(c);
        if (rc) return rc;
    }
    *rank = 0;
    if (a->m == 0 || a->n == 0) return F2_OK;
    if (c.algorithm != F2_ALG_GAUSS && c.k > 8) return fail(F2_INVALID_ARGUMENT, "rank: k must be in 0..8");
    f2_matrix* work = nullptr;
    int rc = f2_matrix_create(a->m, a->n, &work);
    if (rc) return rc;
    if (!(rc = f2_matrix_copy(work, a))) {
        std::vector<uint64_t> p(a->m), q(a->n);
        // the rank is independent of k and of the cutoff: run the engine with the defaults
        const f2_elim_config cp{0, 0, 0.15, F2_ALG_PLS};
        rc = f2_pls_recursive(work, f2_window{0, 0, a->m, a->n}, p.data(), a->m, q.data(), a->n, &cp, rank);
    }
    f2_matrix_destroy(work);
    return rc;
}

}  // extern "C"
