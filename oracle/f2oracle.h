/* TEST INFRASTRUCTURE ONLY (the CPU checker; never linked into the product).
 *
 * C restatement of the reference algorithm on the PLS hot path of
 * arxiv/paper_1006_1744 (`f2lin`, /root/reference/proj).  Host arrays use the
 * reference packing: row-major, stride = ceil(ncols/64) words, bit j of a row in
 * word j/64 at position j%64 (proj/include/f2lin/bitmat.hpp:3-6,31-33).
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * golden vectors of the reference's own tests (tests/golden/) and against the
 * reference sources compiled in place (oracle/_ref, see Makefile).
 */
#ifndef F2ORACLE_H
#define F2ORACLE_H
#include <stddef.h>
#include <stdint.h>

uint64_t f2o_splitmix_next(uint64_t* state);
int f2o_randomize(uint64_t* w, size_t m, size_t n, double density, uint64_t seed);
int f2o_fixed_weight(uint64_t* w, size_t m, size_t n, size_t weight, uint64_t seed);
size_t f2o_gauss_pls(uint64_t* w, size_t m, size_t n, uint64_t* p, uint64_t* q);
void f2o_compress_columns(uint64_t* w, size_t m, size_t n, size_t rank, const uint64_t* q);
size_t f2o_recursive_q(size_t m, size_t n, uint64_t cutoff, size_t rank, const uint64_t* pivcols,
                       uint64_t* q);
void f2o_mul(const uint64_t* a, size_t m, size_t s, const uint64_t* b, size_t n, uint64_t* c);
unsigned f2o_auto_table_bits(size_t dim);
uint64_t f2o_digest(const uint64_t* w, size_t nwords);
int f2o_pls_check(const uint64_t* orig, const uint64_t* packed, size_t m, size_t n, size_t rank,
                  const uint64_t* p, const uint64_t* q);
size_t f2o_gauss_rref(uint64_t* w, size_t m, size_t n);
int f2o_rref_from_pls(uint64_t* w, size_t m, size_t n, size_t rank, const uint64_t* q, size_t qlen);
long f2o_m4ri_rref(uint64_t* w, size_t m, size_t n, unsigned k, int full);
#endif
