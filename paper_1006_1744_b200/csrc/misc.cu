// Streaming kernels around the PLS hot path: seeded generation, fingerprint,
// window extract/insert, row gathers and the final column compression.
#include <cstdint>

#include "f2gpu.cuh"
#include "kernels.cuh"

namespace f2g {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// n bits (<= 64) of row `r` starting at bit b; reads never pass the row stride
__device__ __forceinline__ uint64_t fetch64(const uint64_t* r, int64_t stride, int64_t b) {
    const int64_t w = b >> 6;
    const int s = static_cast<int>(b & 63);
    uint64_t v = r[w] >> s;
    if (s && w + 1 < stride) v |= r[w + 1] << (64 - s);
    return v;
}

}  // namespace

// BitMatrix::randomize (proj/src/bitmat.cpp:136-154): SplitMix64 draw t over the
// real bits in row-major order is mix(seed + (t+1)*golden) (prng.hpp:11-22), so
// every word is generated independently.  bit = (draw >> 11) < threshold.
__global__ void k_randomize(Mat A, uint64_t thr, uint64_t seed) {
    const int64_t nw = (A.n + 63) >> 6;
    const int64_t total = A.m * nw;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / nw, k = idx - i * nw;
        const int nb = static_cast<int>(A.n - 64 * k < 64 ? A.n - 64 * k : 64);
        const uint64_t t0 = static_cast<uint64_t>(i) * static_cast<uint64_t>(A.n) + 64ull * k;
        uint64_t st = seed + (t0 + 1) * 0x9e3779b97f4a7c15ull;
        uint64_t word = 0;
        for (int t = 0; t < nb; ++t) {
            if ((mix64(st) >> 11) < thr) word |= 1ull << t;
            st += 0x9e3779b97f4a7c15ull;
        }
        A.w[i * A.stride + k] = word;
    }
}

// sum of mix(w_i + (i+1)*golden) over the reference packing (i = row*nw + k)
__global__ void k_digest(Mat A, unsigned long long* out) {
    const int64_t nw = (A.n + 63) >> 6;
    const int64_t total = A.m * nw;
    unsigned long long h = 0;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / nw, k = idx - i * nw;
        h += mix64(A.w[i * A.stride + k] + static_cast<uint64_t>(idx + 1) * 0x9e3779b97f4a7c15ull);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

// dst (aligned, dst.m x dst.n) <- window of src at (r0, c0)
__global__ void k_extract(Mat src, int64_t r0, int64_t c0, Mat dst) {
    const int64_t nw = (dst.n + 63) >> 6;
    const int64_t total = dst.m * dst.stride;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / dst.stride, k = idx - i * dst.stride;
        uint64_t v = 0;
        if (k < nw) {
            v = fetch64(src.w + (r0 + i) * src.stride, src.stride, c0 + 64 * k);
            const int64_t rem = dst.n - 64 * k;
            if (rem < 64) v &= (1ull << rem) - 1;
        }
        dst.w[idx] = v;
    }
}

// window of dst at (r0, c0) <- src (aligned); bits outside the window untouched
__global__ void k_insert(Mat dst, int64_t r0, int64_t c0, Mat src) {
    const int64_t jw0 = c0 >> 6, jw1 = (c0 + src.n + 63) >> 6;
    const int64_t nwj = jw1 - jw0;
    const int64_t total = src.m * nwj;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / nwj, j = jw0 + (idx - i * nwj);
        const int64_t off = 64 * j - c0;  // src bit under dst bit 64j
        const uint64_t* sr = src.w + i * src.stride;
        uint64_t v = off >= 0 ? fetch64(sr, src.stride, off) : (sr[0] << (-off));
        uint64_t mask = ~0ull;
        if (off < 0) mask &= ~0ull << (-off);
        const int64_t endb = src.n - off;  // dst-word bit index where the window ends
        if (endb < 64) mask &= endb <= 0 ? 0ull : ((1ull << endb) - 1);
        uint64_t* d = dst.w + (r0 + i) * dst.stride + j;
        *d = (*d & ~mask) | (v & mask);
    }
}

// dst row i (word range [0, nwords)) <- src row rowmap[i]
__global__ void k_gather_rows(Mat dst, Mat src, const int64_t* rowmap, int64_t nrows, int64_t nwords) {
    const int64_t total = nrows * nwords;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / nwords, k = idx - i * nwords;
        dst.w[i * dst.stride + k] = src.w[rowmap[i] * src.stride + k];
    }
}

// Final column compression of a packed PLS result, in closed form.
// compress_columns (perm.cpp:18-21) swaps columns j <-> Q[j] from row j down for
// j < rank.  With the packed layout of an uncompressed PLS (L bits of row i at the
// pivot columns Q[t], t < min(i, rank); pivot row i's leading 1 at Q[i] and S right
// of it; all other columns left of Q[i] zero) the swap sequence works out, per row,
// to: bits [0, min(i,rank)) <- old bits Q[0..); row i < rank: bit i = 1, bits
// (i, Q[i]] = 0, bits > Q[i] unchanged; row i >= rank: everything from rank on 0.
// One CTA per row, the old row staged in SMEM.
__global__ void k_compress(Mat A, int64_t rank, const int64_t* Qp) {
    extern __shared__ uint64_t srow[];
    const int64_t qmax = Qp[rank - 1];
    const int64_t span = (qmax >> 6) + 1;  // words that can change
    for (int64_t i = blockIdx.x; i < A.m; i += gridDim.x) {
        uint64_t* row = A.w + i * A.stride;
        __syncthreads();
        for (int64_t k = threadIdx.x; k < span; k += blockDim.x) srow[k] = row[k];
        __syncthreads();
        const int64_t lim = i < rank ? i : rank;
        const int64_t qi = i < rank ? Qp[i] : -1;
        const int64_t wend = i < rank ? (qi >> 6) + 1 : span;
        for (int64_t k = threadIdx.x; k < wend; k += blockDim.x) {
            const int64_t lo = 64 * k;
            uint64_t v = 0;
            const int64_t ghi = lim < lo + 64 ? lim : lo + 64;
            for (int64_t p = lo; p < ghi; ++p) {
                const int64_t qp = Qp[p];
                v |= ((srow[qp >> 6] >> (qp & 63)) & 1ull) << (p - lo);
            }
            if (i < rank) {
                if (i >= lo && i < lo + 64) v |= 1ull << (i - lo);
                // keep old bits strictly above Q[i]
                const int64_t keep_from = qi + 1;
                if (keep_from < lo + 64) {
                    uint64_t km = keep_from <= lo ? ~0ull : (~0ull << (keep_from - lo));
                    v = (v & ~km) | (srow[k] & km);
                }
            }
            row[k] = v;
        }
    }
}

// compress_columns for an arbitrary transposition vector (perm.cpp:18-21,
// bitmat.cpp:94-110): row i applies swaps j = 0..min(i, rank-1) in order.
__global__ void k_col_swaps(Mat A, int64_t rank, const int64_t* q) {
    extern __shared__ uint64_t srow[];
    const int64_t nw = (A.n + 63) >> 6;
    for (int64_t i = blockIdx.x; i < A.m; i += gridDim.x) {
        uint64_t* row = A.w + i * A.stride;
        __syncthreads();
        for (int64_t k = threadIdx.x; k < nw; k += blockDim.x) srow[k] = row[k];
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t jl = i < rank ? i + 1 : rank;
            for (int64_t j = 0; j < jl; ++j) {
                const int64_t a = j, b = q[j];
                if (a == b) continue;
                const uint64_t va = (srow[a >> 6] >> (a & 63)) & 1ull, vb = (srow[b >> 6] >> (b & 63)) & 1ull;
                if (va != vb) {
                    srow[a >> 6] ^= 1ull << (a & 63);
                    srow[b >> 6] ^= 1ull << (b & 63);
                }
            }
        }
        __syncthreads();
        for (int64_t k = threadIdx.x; k < nw; k += blockDim.x) row[k] = srow[k];
    }
}

static int grid_for(int64_t total, int threads) {
    int64_t g = (total + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    return g < 1 ? 1 : static_cast<int>(g);
}

void launch_randomize(cudaStream_t s, const Mat& A, uint64_t threshold, uint64_t seed) {
    const int64_t total = A.m * ((A.n + 63) >> 6);
    if (total == 0) return;
    k_randomize<<<grid_for(total, 256), 256, 0, s>>>(A, threshold, seed);
}

void launch_digest(cudaStream_t s, const Mat& A, unsigned long long* out) {
    cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    const int64_t total = A.m * ((A.n + 63) >> 6);
    if (total == 0) return;
    k_digest<<<grid_for(total, 256), 256, 0, s>>>(A, out);
}

void launch_extract(cudaStream_t s, const Mat& src, int64_t r0, int64_t c0, const Mat& dst) {
    const int64_t total = dst.m * dst.stride;
    if (total == 0) return;
    k_extract<<<grid_for(total, 256), 256, 0, s>>>(src, r0, c0, dst);
}

void launch_insert(cudaStream_t s, const Mat& dst, int64_t r0, int64_t c0, const Mat& src) {
    if (src.m == 0 || src.n == 0) return;
    const int64_t total = src.m * (((c0 + src.n + 63) >> 6) - (c0 >> 6));
    k_insert<<<grid_for(total, 256), 256, 0, s>>>(dst, r0, c0, src);
}

// dst[i][j] = src[r-1-i][r-1-j] for an r x r bit matrix: a unit upper triangular U becomes
// the unit lower triangular R U R, so U^{-1} B = R (R U R)^{-1} R B runs on the lower solver
__global__ void k_reverse_square(Mat dst, Mat src, int64_t r) {
    const int64_t nw = (r + 63) >> 6, total = r * nw;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / nw, w = idx - i * nw;
        const uint64_t* srow = src.w + (r - 1 - i) * src.stride;
        uint64_t v = 0;
        for (int b = 0; b < 64; ++b) {
            const int64_t j = 64 * w + b;
            if (j >= r) break;
            const int64_t sj = r - 1 - j;
            v |= ((srow[sj >> 6] >> (sj & 63)) & 1ull) << b;
        }
        dst.w[i * dst.stride + w] = v;
    }
}

void launch_reverse_square(cudaStream_t s, const Mat& dst, const Mat& src, int64_t r) {
    const int64_t total = r * ((r + 63) >> 6);
    if (total == 0) return;
    k_reverse_square<<<grid_for(total, 256), 256, 0, s>>>(dst, src, r);
}

void launch_gather_rows(cudaStream_t s, const Mat& dst, const Mat& src, const int64_t* rowmap, int64_t nrows,
                        int64_t nwords) {
    const int64_t total = nrows * nwords;
    if (total == 0) return;
    k_gather_rows<<<grid_for(total, 256), 256, 0, s>>>(dst, src, rowmap, nrows, nwords);
}

void launch_compress(cudaStream_t s, const Mat& A, int64_t rank, const int64_t* Qp, int nsm) {
    if (rank == 0 || A.m == 0) return;
    const int64_t g = A.m < 8 * nsm ? A.m : 8 * nsm;
    const size_t smem = sizeof(uint64_t) * A.stride;
    k_compress<<<static_cast<int>(g), 256, smem, s>>>(A, rank, Qp);
}

void launch_col_swaps(cudaStream_t s, const Mat& A, int64_t rank, const int64_t* q, int nsm) {
    if (rank == 0 || A.m == 0) return;
    const int64_t g = A.m < 8 * nsm ? A.m : 8 * nsm;
    const size_t smem = sizeof(uint64_t) * A.stride;
    k_col_swaps<<<static_cast<int>(g), 128, smem, s>>>(A, rank, q);
}

void setup_misc_kernels() {
    cudaFuncSetAttribute(k_compress, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_col_swaps, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace f2g

namespace f2g {

// rref_from_pls, step 1 (pls.cpp:137-138 with pls_echelon_factor, gauss.cpp:74-83):
// row t < rank becomes S row t in original column order (1 at q[t], the packed bits
// right of it, nothing left of it); rows >= rank become zero.
__global__ void k_rref_prepare(Mat A, int64_t rank, const int64_t* Qp) {
    const int64_t nw = (A.n + 63) >> 6;
    const int64_t total = A.m * nw;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / nw, k = idx - i * nw;
        uint64_t* wp = A.w + i * A.stride + k;
        if (i >= rank) {
            *wp = 0;
            continue;
        }
        const int64_t q = Qp[i], lo = 64 * k;
        uint64_t v = *wp;
        if (q >= lo + 64) v = 0;
        else if (q >= lo) {
            const int b = static_cast<int>(q - lo);
            v = (b == 63 ? 0ull : (v & (~0ull << (b + 1)))) | (1ull << b);
        }
        *wp = v;
    }
}

// Coefficients of the backward substitution, row- and column-reversed so the
// lower-triangular solver applies: Lrev[t'][l'] = S[rank-1-t'] at column q[rank-1-l'].
// One CTA per output row, the S row staged in SMEM.
__global__ void k_rref_coeffs(Mat S, int64_t rank, const int64_t* Qp, Mat Lrev) {
    extern __shared__ uint64_t srow[];
    const int64_t nws = (S.n + 63) >> 6, nwl = (rank + 63) >> 6;
    for (int64_t tp = blockIdx.x; tp < rank; tp += gridDim.x) {
        const uint64_t* row = S.w + (rank - 1 - tp) * S.stride;
        __syncthreads();
        for (int64_t k = threadIdx.x; k < nws; k += blockDim.x) srow[k] = row[k];
        __syncthreads();
        for (int64_t w = threadIdx.x; w < nwl; w += blockDim.x) {
            uint64_t v = 0;
            const int64_t l0 = 64 * w;
            const int nb = static_cast<int>(rank - l0 < 64 ? rank - l0 : 64);
            for (int b = 0; b < nb; ++b) {
                const int64_t col = Qp[rank - 1 - (l0 + b)];
                v |= ((srow[col >> 6] >> (col & 63)) & 1ull) << b;
            }
            Lrev.w[tp * Lrev.stride + w] = v;
        }
    }
}

void launch_rref_prepare(cudaStream_t s, const Mat& A, int64_t rank, const int64_t* Qp) {
    const int64_t total = A.m * ((A.n + 63) >> 6);
    if (total == 0) return;
    int64_t g = (total + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    k_rref_prepare<<<static_cast<int>(g), 256, 0, s>>>(A, rank, Qp);
}

void launch_rref_coeffs(cudaStream_t s, const Mat& S, int64_t rank, const int64_t* Qp, const Mat& Lrev, int nsm) {
    if (rank == 0) return;
    const int64_t g = rank < 8 * nsm ? rank : 8 * nsm;
    k_rref_coeffs<<<static_cast<int>(g), 256, sizeof(uint64_t) * S.stride, s>>>(S, rank, Qp, Lrev);
}

// M4RI's non-full echelon form (m4ri_rref(a, k, false), m4ri.cpp:68-87) from U: within
// each block of consecutive pivots that one gauss_submatrix call forms (m4ri.cpp:45-67),
// the block's rows are reduced against each other on the block's pivot columns (RREF
// inside the block only).  One CTA per block, rows bottom-up; a row's coefficients come
// from its unreduced bits (the reduced later rows are zero on each other's pivots).
__global__ void __launch_bounds__(256) k_block_backsub(Mat U, const int64_t* __restrict__ bstart,
                                                       const int64_t* __restrict__ Qp, int64_t nblocks) {
    __shared__ uint32_t s_mask;
    const int64_t nw = (U.n + 63) >> 6;
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int64_t t0 = bstart[b], t1 = bstart[b + 1];
        const int64_t w0 = Qp[t0] >> 6;  // every row of the block is zero left of its first pivot
        for (int64_t t = t1 - 2; t >= t0; --t) {
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t mk = 0;
                for (int64_t u = t + 1; u < t1; ++u) {
                    const int64_t q = Qp[u];
                    if ((U.w[t * U.stride + (q >> 6)] >> (q & 63)) & 1ull) mk |= 1u << (u - t - 1);
                }
                s_mask = mk;
            }
            __syncthreads();
            const uint32_t mk = s_mask;
            if (!mk) continue;
            for (int64_t k = w0 + threadIdx.x; k < nw; k += blockDim.x) {
                uint64_t v = U.w[t * U.stride + k];
                for (uint32_t x = mk; x; x &= x - 1) v ^= U.w[(t + 1 + __ffs(x) - 1) * U.stride + k];
                U.w[t * U.stride + k] = v;
            }
        }
    }
}

void launch_block_backsub(cudaStream_t s, const Mat& U, const int64_t* bstart, const int64_t* Qp, int64_t nblocks,
                          int nsm) {
    if (nblocks <= 0) return;
    const int64_t g = nblocks < 8 * nsm ? nblocks : 8 * nsm;
    k_block_backsub<<<static_cast<int>(g), 256, 0, s>>>(U, bstart, Qp, nblocks);
}

void setup_rref_kernels() {
    cudaFuncSetAttribute(k_rref_coeffs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}


}  // namespace f2g
