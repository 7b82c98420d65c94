// TEST HARNESS for integration/f2lin_gpu_adapter.hpp: a reference BitMatrix built from
// host words, decomposed through the adapter (and so through libf2gpu.so), written
// back.  tests/test_gpu_integration.py compares the result with the reference's own
// pls_recursive / mmpf_pls (oracle/_ref/libf2ref.so).
#include <cstring>

#include "f2lin_gpu_adapter.hpp"

extern "C" int adapter_pls(int recursive, uint64_t* w, size_t m, size_t n, uint64_t cutoff, unsigned k, uint64_t* p,
                           uint64_t* q, uint64_t* rank) {
    try {
        f2lin::BitMatrix a(m, n);
        for (size_t i = 0; i < m; ++i) std::memcpy(a.row(i), w + i * a.stride(), a.stride() * 8);
        f2lin::Permutation P, Q;
        f2lin::EliminationConfig cfg;
        cfg.k = k;
        cfg.cutoff_bytes = cutoff;
        *rank = recursive ? f2lin_gpu::pls_recursive_gpu(a, P, Q, cfg) : f2lin_gpu::mmpf_pls_gpu(a, P, Q, k);
        for (size_t i = 0; i < m; ++i) std::memcpy(w + i * a.stride(), a.row(i), a.stride() * 8);
        for (size_t i = 0; i < m; ++i) p[i] = P[i];
        for (size_t j = 0; j < n; ++j) q[j] = Q[j];
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (...) {
        return 9;
    }
}
