/* TEST INFRASTRUCTURE ONLY — CPU checker for the GPU PLS engine.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 * See f2oracle.h for the packing convention; every function cites the
 * reference lines (under /root/reference/proj) it restates.
 */
#include "f2oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define WORDS(n) (((n) + 63) / 64)
#define GET(w, s, i, j) (((w)[(i) * (s) + (j) / 64] >> ((j) % 64)) & 1u)

/* SplitMix64 — include/f2lin/prng.hpp:11-22 */
uint64_t f2o_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* BitMatrix::randomize — src/bitmat.cpp:136-154: one draw per real bit,
 * row-major, padding consumes none; bit = (draw>>11) < llround(d*2^53). */
int f2o_randomize(uint64_t* w, size_t m, size_t n, double density, uint64_t seed) {
    if (!(density >= 0.0 && density <= 1.0)) return 1;
    uint64_t thr = (uint64_t)llround(density * 9007199254740992.0);
    uint64_t st = seed;
    size_t s = WORDS(n);
    for (size_t i = 0; i < m; ++i)
        for (size_t k = 0; k < s; ++k) {
            size_t nb = n - k * 64 < 64 ? n - k * 64 : 64;
            uint64_t word = 0;
            for (size_t t = 0; t < nb; ++t)
                if ((f2o_splitmix_next(&st) >> 11) < thr) word |= 1ull << t;
            w[i * s + k] = word;
        }
    return 0;
}

/* Config-5 generator (no reference counterpart; SURVEY.md §8d defines it):
 * one SplitMix64(seed) stream; per row draw next() % n and reject duplicates
 * until `weight` distinct columns are set.  n need not be a power of two here,
 * the draw is then slightly biased — the contract is the stream, not the law. */
int f2o_fixed_weight(uint64_t* w, size_t m, size_t n, size_t weight, uint64_t seed) {
    if (weight > n) return 1;
    uint64_t st = seed;
    size_t s = WORDS(n);
    memset(w, 0, m * s * 8);
    for (size_t i = 0; i < m; ++i) {
        uint64_t* row = w + i * s;
        size_t got = 0;
        while (got < weight) {
            size_t j = (size_t)(f2o_splitmix_next(&st) % n);
            uint64_t bit = 1ull << (j % 64);
            if (row[j / 64] & bit) continue;
            row[j / 64] |= bit;
            ++got;
        }
    }
    return 0;
}

/* col_swap_range — src/bitmat.cpp:94-110 (element-wise restatement) */
static void col_swap_from(uint64_t* w, size_t s, size_t m, size_t a, size_t b, size_t r0) {
    for (size_t i = r0; i < m; ++i) {
        uint64_t* row = w + i * s;
        uint64_t va = (row[a / 64] >> (a % 64)) & 1u, vb = (row[b / 64] >> (b % 64)) & 1u;
        if (va != vb) {
            row[a / 64] ^= 1ull << (a % 64);
            row[b / 64] ^= 1ull << (b % 64);
        }
    }
}

/* compress_columns_span — src/perm.cpp:18-21: for j < rank ascending, swap
 * columns j and q[j] from row j down. */
void f2o_compress_columns(uint64_t* w, size_t m, size_t n, size_t rank, const uint64_t* q) {
    size_t s = WORDS(n);
    for (size_t j = 0; j < rank; ++j)
        if (q[j] != j) col_swap_from(w, s, m, j, (size_t)q[j], j);
}

/* gauss_pls — src/gauss.cpp:26-55.  Pivot = leftmost column with a nonzero at
 * or below row r, first such row in the current order (:33-40); record
 * P[r]=i, Q[r]=j (:42-43); swap rows (:44); clear below starting one column
 * right of the pivot so the L bit stays (:47-49); compress (:53). */
size_t f2o_gauss_pls(uint64_t* w, size_t m, size_t n, uint64_t* p, uint64_t* q) {
    size_t s = WORDS(n);
    for (size_t i = 0; i < m; ++i) p[i] = i;
    for (size_t j = 0; j < n; ++j) q[j] = j;
    size_t r = 0, c = 0;
    uint64_t* tmp = (uint64_t*)malloc(s * 8 + 8);
    while (r < m && c < n) {
        size_t pi = m, pj = n;
        for (size_t j = c; j < n && pj == n; ++j)
            for (size_t i = r; i < m; ++i)
                if (GET(w, s, i, j)) {
                    pi = i;
                    pj = j;
                    break;
                }
        if (pj == n) break;
        p[r] = pi;
        q[r] = pj;
        if (pi != r) {
            memcpy(tmp, w + r * s, s * 8);
            memcpy(w + r * s, w + pi * s, s * 8);
            memcpy(w + pi * s, tmp, s * 8);
        }
        if (pj + 1 < n) {
            size_t b = pj + 1, w0 = b / 64;
            uint64_t m0 = ~0ull << (b % 64);
            const uint64_t* src = w + r * s;
            for (size_t l = r + 1; l < m; ++l) {
                uint64_t* dst = w + l * s;
                if (!((dst[pj / 64] >> (pj % 64)) & 1u)) continue;
                dst[w0] ^= src[w0] & m0;
                for (size_t k = w0 + 1; k < s; ++k) dst[k] ^= src[k];
            }
        }
        r = r + 1;
        c = pj + 1;
    }
    free(tmp);
    f2o_compress_columns(w, m, n, r, q);
    return r;
}

/* Replay of pls_recursive_impl's Q bookkeeping — src/pls.cpp:63-103.  Q is a
 * pure function of (m, n, cutoff, global pivot columns): leaf rule :71
 * (n <= 64 || rows*ceil(cols/8) <= cutoff, leaf = mmpf_pls whose Q is the
 * identity with the pivot prefix, mmpf.cpp:87-88,37), cut :74-75, merge
 * :96-98 (which leaves stale q1[t]+n0 entries behind the rank). */
static void replay(size_t m, size_t n, uint64_t cutoff, const uint64_t* piv, size_t npiv,
                   uint64_t* q) {
    for (size_t j = 0; j < n; ++j) q[j] = j;
    if (m == 0 || n == 0) return;
    if (n <= 64 || (uint64_t)m * ((n + 7) / 8) <= cutoff) {
        for (size_t t = 0; t < npiv; ++t) q[t] = piv[t];
        return;
    }
    size_t n0 = ((n / 2 + 63) / 64) * 64;
    if (n0 >= n) n0 = n / 2;
    size_t r0 = 0;
    while (r0 < npiv && piv[r0] < n0) ++r0;
    replay(m, n0, cutoff, piv, r0, q);
    size_t r1 = npiv - r0;
    uint64_t* sub = (uint64_t*)malloc((r1 ? r1 : 1) * 8);
    for (size_t t = 0; t < r1; ++t) sub[t] = piv[r0 + t] - n0;
    replay(m - r0, n - n0, cutoff, sub, r1, q + n0);
    free(sub);
    for (size_t i = n0; i < n; ++i) q[i] += n0;
    for (size_t t = 0; t < r1; ++t) q[r0 + t] = q[n0 + t];
}

size_t f2o_recursive_q(size_t m, size_t n, uint64_t cutoff, size_t rank, const uint64_t* pivcols,
                       uint64_t* q) {
    replay(m, n, cutoff, pivcols, rank, q);
    return rank;
}

/* mul_naive — src/mul.cpp:73-88 */
void f2o_mul(const uint64_t* a, size_t m, size_t s, const uint64_t* b, size_t n, uint64_t* c) {
    size_t sa = WORDS(s), sb = WORDS(n);
    memset(c, 0, m * sb * 8);
    for (size_t i = 0; i < m; ++i)
        for (size_t l = 0; l < s; ++l)
            if (GET(a, sa, i, l))
                for (size_t k = 0; k < sb; ++k) c[i * sb + k] ^= b[l * sb + k];
}

/* auto_table_bits — src/mul.cpp:9-14 */
unsigned f2o_auto_table_bits(size_t dim) {
    if (dim < 2) return 1;
    unsigned lg = 0;
    while ((dim >> (lg + 1)) != 0) ++lg;
    if (lg <= 3) return 1;
    return lg - 2 > 8 ? 8 : lg - 2;
}

/* Order-sensitive 64-bit fingerprint of a word array (ours, for golden
 * fixtures of the full-size configs): sum of splitmix(w_i + (i+1)*golden). */
uint64_t f2o_digest(const uint64_t* w, size_t nwords) {
    uint64_t h = 0;
    for (size_t i = 0; i < nwords; ++i) {
        uint64_t z = w[i] + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        h += z ^ (z >> 31);
    }
    return h;
}

/* pls_verify — src/gauss.cpp:63-91 (pls_unit_lower / pls_echelon_factor /
 * apply_rows_inverse): returns 1 iff P^-1 * L * S == orig. */
int f2o_pls_check(const uint64_t* orig, const uint64_t* packed, size_t m, size_t n, size_t rank,
                  const uint64_t* p, const uint64_t* q) {
    size_t s = WORDS(n);
    uint64_t* srow = (uint64_t*)calloc(rank * s + 1, 8);
    uint64_t* out = (uint64_t*)calloc(m * s + 1, 8);
    for (size_t t = 0; t < rank; ++t) { /* S row t: 1 at q[t], copy packed right of it */
        size_t piv = (size_t)q[t];
        srow[t * s + piv / 64] |= 1ull << (piv % 64);
        for (size_t j = piv + 1; j < n; ++j)
            if (GET(packed, s, t, j)) srow[t * s + j / 64] |= 1ull << (j % 64);
    }
    for (size_t i = 0; i < m; ++i) { /* (L*S) row i */
        size_t upto = i < rank ? i : rank;
        for (size_t j = 0; j < upto; ++j)
            if (GET(packed, s, i, j))
                for (size_t k = 0; k < s; ++k) out[i * s + k] ^= srow[j * s + k];
        if (i < rank)
            for (size_t k = 0; k < s; ++k) out[i * s + k] ^= srow[i * s + k];
    }
    for (size_t i = m; i-- > 0;) /* apply_rows_inverse: descending swaps */
        if (p[i] != i)
            for (size_t k = 0; k < s; ++k) {
                uint64_t t = out[i * s + k];
                out[i * s + k] = out[p[i] * s + k];
                out[p[i] * s + k] = t;
            }
    int ok = memcmp(out, orig, m * s * 8) == 0;
    free(srow);
    free(out);
    return ok;
}

/* gauss_rref — src/gauss.cpp:7-23: column by column, first row >= r with a 1,
 * swap it up, clear the column in every other row. */
size_t f2o_gauss_rref(uint64_t* w, size_t m, size_t n) {
    size_t s = WORDS(n), r = 0;
    for (size_t c = 0; c < n && r < m; ++c) {
        size_t piv = m;
        for (size_t i = r; i < m; ++i)
            if (GET(w, s, i, c)) {
                piv = i;
                break;
            }
        if (piv == m) continue;
        for (size_t k = 0; k < s; ++k) {
            uint64_t t = w[r * s + k];
            w[r * s + k] = w[piv * s + k];
            w[piv * s + k] = t;
        }
        for (size_t i = 0; i < m; ++i)
            if (i != r && GET(w, s, i, c))
                for (size_t k = 0; k < s; ++k) w[i * s + k] ^= w[r * s + k];
        ++r;
    }
    return r;
}

static void col_swap_rows(uint64_t* w, size_t s, size_t r0, size_t r1, size_t a, size_t b) {
    for (size_t i = r0; i < r1; ++i) {
        uint64_t* row = w + i * s;
        uint64_t va = (row[a / 64] >> (a % 64)) & 1u, vb = (row[b / 64] >> (b % 64)) & 1u;
        if (va != vb) {
            row[a / 64] ^= 1ull << (a % 64);
            row[b / 64] ^= 1ull << (b % 64);
        }
    }
}

/* rref_from_pls — src/pls.cpp:128-155, step for step: validation (:130-135);
 * zero the L storage and the rows >= rank (:137-138); complete the column swaps
 * over the rows above (:145-146); unit upper triangular solve of the top block
 * against columns rank..n (:148-149, trsm_upper_left_unit mul.cpp:133-155,
 * restated as plain back substitution, bottom row first); identity pivot block
 * (:151); undo the swaps in reverse (:153-154).  Returns 1 on invalid_argument. */
int f2o_rref_from_pls(uint64_t* w, size_t m, size_t n, size_t rank, const uint64_t* q, size_t qlen) {
    size_t s = WORDS(n);
    if (rank > m || rank > n || qlen < rank) return 1;
    for (size_t t = 0; t < rank; ++t)
        if (q[t] >= n || q[t] < t || (t > 0 && q[t] <= q[t - 1])) return 1;
    for (size_t i = 1; i < m; ++i)
        for (size_t j = 0; j < (i < rank ? i : rank); ++j) w[i * s + j / 64] &= ~(1ull << (j % 64));
    for (size_t i = rank; i < m; ++i)
        for (size_t k = 0; k < s; ++k) w[i * s + k] = 0;
    for (size_t j = 0; j < rank; ++j)
        if (q[j] != j) col_swap_rows(w, s, 0, j, j, (size_t)q[j]);
    if (rank > 0 && rank < n) {
        /* row u -= sum_{v>u} T[u][v] * row v over columns >= rank, v descending */
        for (size_t u = rank; u-- > 0;)
            for (size_t v = u + 1; v < rank; ++v)
                if (GET(w, s, u, v))
                    for (size_t j = rank; j < n; ++j)
                        if (GET(w, s, v, j)) w[u * s + j / 64] ^= 1ull << (j % 64);
    }
    for (size_t u = 0; u < rank; ++u)
        for (size_t j = u + 1; j < rank; ++j) w[u * s + j / 64] &= ~(1ull << (j % 64));
    for (size_t j = rank; j-- > 0;)
        if (q[j] != j) col_swap_rows(w, s, 0, rank, j, (size_t)q[j]);
    return 0;
}

/* row i ^= row src over columns [from, n) — BitMatrix::row_add, include/f2lin/bitmat.hpp */
static void row_add_from(uint64_t* w, size_t s, size_t n, size_t i, size_t src, size_t from) {
    if (from >= n) return;
    size_t k0 = from / 64;
    uint64_t first = ~0ull << (from % 64);
    w[i * s + k0] ^= w[src * s + k0] & first;
    for (size_t k = k0 + 1; k < WORDS(n); ++k) w[i * s + k] ^= w[src * s + k];
}

static void row_swap_full(uint64_t* w, size_t s, size_t a, size_t b) {
    if (a == b) return;
    for (size_t k = 0; k < s; ++k) {
        uint64_t t = w[a * s + k];
        w[a * s + k] = w[b * s + k];
        w[b * s + k] = t;
    }
}

/* gauss_submatrix — src/m4ri.cpp:45-67: RREF of the k-column block at (r, c), pivots
 * searched in rows [r, r_end) with lazy clearing of the block's earlier columns. */
static unsigned gauss_submatrix(uint64_t* w, size_t s, size_t n, size_t r, size_t c, unsigned k, size_t r_end) {
    size_t r_s = r;
    for (size_t j = c; j < c + k; ++j) {
        int found = 0;
        for (size_t i = r_s; i < r_end; ++i) {
            for (size_t l = 0; l < j - c; ++l)
                if (GET(w, s, i, c + l)) row_add_from(w, s, n, i, r + l, c + l);
            if (GET(w, s, i, j)) {
                row_swap_full(w, s, i, r_s);
                for (size_t l = r; l < r_s; ++l)
                    if (GET(w, s, l, j)) row_add_from(w, s, n, l, r_s, j);
                ++r_s;
                found = 1;
                break;
            }
        }
        if (!found) break;
    }
    return (unsigned)(r_s - r);
}

/* m4ri_rref — src/m4ri.cpp:68-87.  The table step (make_table :11-26 +
 * add_rows_from_table :28-38) adds, to every row outside the block, the combination
 * of the block's pivot rows that clears its kbar block bits; the block rows are the
 * identity on the block's (consecutive) pivot columns, so that combination is the
 * sum of the pivot rows whose column bit is set.  Returns the rank, or -1 for k > 8. */
long f2o_m4ri_rref(uint64_t* w, size_t m, size_t n, unsigned k, int full) {
    if (m == 0 || n == 0) return 0;
    if (k > 8) return -1;
    size_t s = WORDS(n);
    unsigned k0 = k ? k : f2o_auto_table_bits(m < n ? m : n);
    size_t r = 0, c = 0;
    while (r < m && c < n) {
        unsigned kc = (unsigned)(n - c < k0 ? n - c : k0);
        unsigned kbar = gauss_submatrix(w, s, n, r, c, kc, m);
        if (kbar > 0) {
            for (size_t i = 0; i < m; ++i) {
                if (i >= r && i < r + kbar) continue;
                if (i < r && !full) continue;
                for (unsigned b = 0; b < kbar; ++b)
                    if (GET(w, s, i, c + b)) row_add_from(w, s, n, i, r + b, c);
            }
            r += kbar;
            c += kbar;
        }
        if (kbar != kc) ++c;
    }
    return (long)r;
}
