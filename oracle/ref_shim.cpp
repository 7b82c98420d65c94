// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the *unmodified* reference library sources compiled from
// /root/reference/proj/src (see oracle/Makefile).  It lets the parity tests and
// bench.py's `--impl reference` arm drive the reference's own entry points:
//   mmpf_pls            (proj/include/f2lin/mmpf.hpp:35-37, proj/src/mmpf.cpp:118-133)
//   pls_recursive       (proj/include/f2lin/pls.hpp:42-47, proj/src/pls.cpp:105-126)
//   gauss_pls           (proj/src/gauss.cpp:26-55)
//   rref_from_pls       (proj/src/pls.cpp:128-161)
//   gauss_rref          (proj/src/gauss.cpp:7-23)
//   m4ri_rref           (proj/include/f2lin/m4ri.hpp:41, proj/src/m4ri.cpp:68-87)
//   hybrid_rref, rank   (proj/include/f2lin/pls.hpp:61-64, proj/src/pls.cpp:163-216)
//   io::read/write_matrix, read/write_permutation (proj/src/io.cpp)
//   mul_m4rm / addmul   (proj/src/mul.cpp:90-107)
//   trsm_*_left_unit    (proj/src/mul.cpp:109-157)
//   BitMatrix::randomize(proj/src/bitmat.cpp:136-154)
//   Permutation::apply_rows[_inverse], compress_columns (proj/src/perm.cpp:25-60)
// Host arrays use the reference's packing: row-major, stride = ceil(ncols/64)
// 64-bit words, LSB = lowest column (bitmat.hpp:3-6).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include <f2lin/gauss.hpp>
#include <f2lin/io.hpp>
#include <filesystem>
#include <f2lin/m4ri.hpp>
#include <f2lin/mmpf.hpp>
#include <f2lin/mul.hpp>
#include <f2lin/perm.hpp>
#include <f2lin/pls.hpp>

using namespace f2lin;

namespace {

BitMatrix load(const uint64_t* w, size_t m, size_t n) {
    BitMatrix a(m, n);
    size_t s = a.stride();
    for (size_t i = 0; i < m; ++i) std::memcpy(a.row(i), w + i * s, s * 8);
    return a;
}

void store(const BitMatrix& a, uint64_t* w) {
    size_t s = a.stride();
    for (size_t i = 0; i < a.nrows(); ++i) std::memcpy(w + i * s, a.row(i), s * 8);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const io::FormatError&) {
        return 6;
    } catch (...) {
        return 9;
    }
}

Permutation perm_of(const uint64_t* v, size_t len) {
    Permutation p = Permutation::identity(len);
    for (size_t i = 0; i < len; ++i) p[i] = static_cast<std::size_t>(v[i]);
    return p;
}

} // namespace

extern "C" {

int ref_randomize(uint64_t* w, size_t m, size_t n, double density, uint64_t seed) {
    return guard([&] {
        BitMatrix a(m, n);
        a.randomize(density, seed);
        store(a, w);
    });
}

int ref_mmpf_pls(uint64_t* w, size_t m, size_t n, unsigned k, uint64_t* p, uint64_t* q,
                 uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        Permutation P, Q;
        *rank = mmpf_pls(a, P, Q, k);
        store(a, w);
        for (size_t i = 0; i < m; ++i) p[i] = P[i];
        for (size_t i = 0; i < n; ++i) q[i] = Q[i];
    });
}

int ref_pls_recursive(uint64_t* w, size_t m, size_t n, unsigned k, uint64_t cutoff, uint64_t* p,
                      uint64_t* q, uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        Permutation P, Q;
        EliminationConfig cfg;
        cfg.k = k;
        cfg.cutoff_bytes = cutoff;
        *rank = pls_recursive(a, P, Q, cfg);
        store(a, w);
        for (size_t i = 0; i < m; ++i) p[i] = P[i];
        for (size_t i = 0; i < n; ++i) q[i] = Q[i];
    });
}

int ref_gauss_pls(uint64_t* w, size_t m, size_t n, uint64_t* p, uint64_t* q, uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        Permutation P, Q;
        *rank = gauss_pls(a, P, Q);
        store(a, w);
        for (size_t i = 0; i < m; ++i) p[i] = P[i];
        for (size_t i = 0; i < n; ++i) q[i] = Q[i];
    });
}

int ref_rref_from_pls(uint64_t* w, size_t m, size_t n, uint64_t rank, const uint64_t* q,
                      size_t qlen) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        std::vector<size_t> qv(q, q + qlen);
        rref_from_pls(a.view(), rank, std::span<const size_t>(qv));
        store(a, w);
    });
}

int ref_m4ri_rref(uint64_t* w, size_t m, size_t n, unsigned k, int full, uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        *rank = m4ri_rref(a, k, full != 0);
        store(a, w);
    });
}

int ref_hybrid_rref(uint64_t* w, size_t m, size_t n, unsigned k, uint64_t cutoff, double threshold,
                    uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        EliminationConfig cfg;
        cfg.k = k;
        cfg.cutoff_bytes = cutoff;
        cfg.hybrid_threshold = threshold;
        *rank = hybrid_rref(a, cfg);
        store(a, w);
    });
}

int ref_rank(const uint64_t* w, size_t m, size_t n, int algorithm, unsigned k, uint64_t cutoff, double threshold,
             uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        EliminationConfig cfg;
        cfg.k = k;
        cfg.cutoff_bytes = cutoff;
        cfg.hybrid_threshold = threshold;
        cfg.algorithm = static_cast<Algorithm>(algorithm);
        *rank = f2lin::rank(a, cfg);
    });
}

int ref_gauss_rref(uint64_t* w, size_t m, size_t n, uint64_t* rank) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        *rank = gauss_rref(a);
        store(a, w);
    });
}

int ref_mul_m4rm(const uint64_t* a, size_t m, size_t s, const uint64_t* b, size_t n, unsigned k,
                 uint64_t* c) {
    return guard([&] {
        BitMatrix A = load(a, m, s), B = load(b, s, n);
        store(mul_m4rm(A, B, k), c);
    });
}

int ref_mul_naive(const uint64_t* a, size_t m, size_t s, const uint64_t* b, size_t n,
                  uint64_t* c) {
    return guard([&] {
        BitMatrix A = load(a, m, s), B = load(b, s, n);
        store(mul_naive(A, B), c);
    });
}

int ref_trsm_lower_left_unit(const uint64_t* l, size_t r, uint64_t* b, size_t n) {
    return guard([&] {
        BitMatrix L = load(l, r, r), B = load(b, r, n);
        trsm_lower_left_unit(L.view(), B.view());
        store(B, b);
    });
}

int ref_trsm_upper_left_unit(const uint64_t* u, size_t r, uint64_t* b, size_t n) {
    return guard([&] {
        BitMatrix U = load(u, r, r), B = load(b, r, n);
        trsm_upper_left_unit(U.view(), B.view());
        store(B, b);
    });
}

size_t ref_default_cutoff_bytes() { return default_cutoff_bytes(); }

unsigned ref_auto_table_bits(size_t dim) { return detail::auto_table_bits(dim); }

// io::write_matrix(path, a, fmt) — fmt 0 ascii, 1 binary
int ref_write_matrix(const char* path, const uint64_t* w, size_t m, size_t n, int fmt) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        io::write_matrix(std::filesystem::path(path), a, fmt ? io::Format::binary : io::Format::ascii);
    });
}

// io::read_matrix(path): dims and format always reported; words copied when they fit
int ref_read_matrix(const char* path, uint64_t* w, size_t cap_words, uint64_t* m, uint64_t* n, int* fmt) {
    return guard([&] {
        io::Format f;
        BitMatrix a = io::read_matrix(std::filesystem::path(path), &f);
        *m = a.nrows();
        *n = a.ncols();
        *fmt = f == io::Format::binary ? 1 : 0;
        if (w && a.nrows() * a.stride() <= cap_words) store(a, w);
    });
}

int ref_write_permutation(const char* path, const uint64_t* p, size_t len) {
    return guard([&] {
        Permutation q = Permutation::identity(len);
        for (size_t i = 0; i < len; ++i) q[i] = p[i];
        io::write_permutation(std::filesystem::path(path), q);
    });
}

int ref_read_permutation(const char* path, uint64_t* p, size_t cap, size_t* len) {
    return guard([&] {
        Permutation q = io::read_permutation(std::filesystem::path(path));
        *len = q.size();
        if (p && q.size() <= cap)
            for (size_t i = 0; i < q.size(); ++i) p[i] = q[i];
    });
}

int ref_apply_rows(uint64_t* w, size_t m, size_t n, const uint64_t* v, size_t len, int inverse) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        const Permutation p = perm_of(v, len);
        if (inverse) p.apply_rows_inverse(a);
        else p.apply_rows(a);
        store(a, w);
    });
}

int ref_compress_columns(uint64_t* w, size_t m, size_t n, size_t rank, const uint64_t* q, size_t qlen) {
    return guard([&] {
        BitMatrix a = load(w, m, n);
        compress_columns(a, rank, perm_of(q, qlen));
        store(a, w);
    });
}

} // extern "C"
