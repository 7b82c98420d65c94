// Reference-side binding: drop-ins for f2lin's decomposition entry points that route
// through the B200 engine's C ABI (include/f2lin_gpu.h).  A caller of the reference
// keeps its BitMatrix / Permutation / EliminationConfig types; the BitMatrix word
// layout is the reference's own (bitmat.hpp:3-6), so rows are passed verbatim.
//
//   pls_recursive_gpu(BitMatrix&, Permutation&, Permutation&, cfg)  <-> pls_recursive  pls.hpp:44-45
//   mmpf_pls_gpu(BitMatrix&, Permutation&, Permutation&, k)         <-> mmpf_pls       mmpf.hpp:36
//
// Errors are rethrown as the reference throws them (invalid_argument, out_of_range).
// Built and run against the reference itself by tests/test_gpu_integration.py
// (integration/adapter_check.cpp, oracle/Makefile target `adapter`).
#pragma once

#include <cstdint>
#include <stdexcept>

#include <f2lin/mmpf.hpp>
#include <f2lin/pls.hpp>

#include "../include/f2lin_gpu.h"

namespace f2lin_gpu {

inline void rethrow(int rc) {
    if (rc == F2_OK) return;
    if (rc == F2_INVALID_ARGUMENT) throw std::invalid_argument(f2_last_error());
    if (rc == F2_OUT_OF_RANGE) throw std::out_of_range(f2_last_error());
    throw std::runtime_error(f2_last_error());
}

static_assert(sizeof(std::size_t) == sizeof(uint64_t), "Permutation slots are passed as uint64_t");

inline std::size_t pls_recursive_gpu(f2lin::BitMatrix& a, f2lin::Permutation& p, f2lin::Permutation& q,
                                     const f2lin::EliminationConfig& cfg = {}) {
    p = f2lin::Permutation::identity(a.nrows());
    q = f2lin::Permutation::identity(a.ncols());
    const f2_elim_config c{cfg.k, cfg.cutoff_bytes, cfg.hybrid_threshold, static_cast<int>(cfg.algorithm)};
    uint64_t rank = 0;
    rethrow(f2_pls_recursive_host(a.nrows() ? a.row(0) : nullptr, a.nrows(), a.ncols(), a.stride(),
                                  reinterpret_cast<uint64_t*>(p.slots().data()),
                                  reinterpret_cast<uint64_t*>(q.slots().data()), &c, &rank));
    return static_cast<std::size_t>(rank);
}

inline std::size_t mmpf_pls_gpu(f2lin::BitMatrix& a, f2lin::Permutation& p, f2lin::Permutation& q,
                                unsigned k = 0) {
    p = f2lin::Permutation::identity(a.nrows());
    q = f2lin::Permutation::identity(a.ncols());
    uint64_t rank = 0;
    rethrow(f2_mmpf_pls_host(a.nrows() ? a.row(0) : nullptr, a.nrows(), a.ncols(), a.stride(),
                             reinterpret_cast<uint64_t*>(p.slots().data()),
                             reinterpret_cast<uint64_t*>(q.slots().data()), k, &rank));
    return static_cast<std::size_t>(rank);
}

}  // namespace f2lin_gpu
