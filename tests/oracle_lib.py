"""TEST INFRASTRUCTURE: ctypes bindings to the two CPU checkers.

* ``Oracle``  -> oracle/_build/libf2oracle.so (our C restatement, travels to the GPU box)
* ``RefLib``  -> oracle/_ref/libf2ref.so     (the reference's own sources compiled in
                 place by oracle/Makefile; built here, travels as a prebuilt .so)

Matrices on this side are numpy uint64 arrays of shape (m, ceil(n/64)) in the
reference packing (bitmat.hpp:3-6).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libf2oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libf2ref.so")

u64p = C.POINTER(C.c_uint64)
sz = C.c_size_t


def words(n: int) -> int:
    return (n + 63) // 64


def ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(u64p)


def digest(w: np.ndarray) -> int:
    """Same fingerprint as f2o_digest, vectorised (chunks keep temporaries small)."""
    flat = np.ascontiguousarray(w).reshape(-1)
    h = np.uint64(0)
    g = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        for s in range(0, flat.size, 1 << 22):
            z = flat[s:s + (1 << 22)] + (np.arange(s + 1, s + 1 + min(1 << 22, flat.size - s), dtype=np.uint64) * g)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            h = h + z.sum(dtype=np.uint64)
    return int(h)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.f2o_randomize.argtypes = [u64p, sz, sz, C.c_double, C.c_uint64]
        L.f2o_fixed_weight.argtypes = [u64p, sz, sz, sz, C.c_uint64]
        L.f2o_gauss_pls.argtypes = [u64p, sz, sz, u64p, u64p]
        L.f2o_gauss_pls.restype = sz
        L.f2o_compress_columns.argtypes = [u64p, sz, sz, sz, u64p]
        L.f2o_recursive_q.argtypes = [sz, sz, C.c_uint64, sz, u64p, u64p]
        L.f2o_recursive_q.restype = sz
        L.f2o_mul.argtypes = [u64p, sz, sz, u64p, sz, u64p]
        L.f2o_auto_table_bits.argtypes = [sz]
        L.f2o_auto_table_bits.restype = C.c_uint
        L.f2o_digest.argtypes = [u64p, sz]
        L.f2o_digest.restype = C.c_uint64
        L.f2o_pls_check.argtypes = [u64p, u64p, sz, sz, sz, u64p, u64p]
        L.f2o_pls_check.restype = C.c_int
        L.f2o_gauss_rref.argtypes = [u64p, sz, sz]
        L.f2o_gauss_rref.restype = sz
        L.f2o_rref_from_pls.argtypes = [u64p, sz, sz, sz, u64p, sz]
        L.f2o_rref_from_pls.restype = C.c_int
        L.f2o_m4ri_rref.argtypes = [u64p, sz, sz, C.c_uint, C.c_int]
        L.f2o_m4ri_rref.restype = C.c_long

    def randomize(self, m, n, density, seed):
        w = np.zeros((m, words(n)), dtype=np.uint64)
        assert self.lib.f2o_randomize(ptr(w), m, n, density, seed) == 0
        return w

    def fixed_weight(self, m, n, weight, seed):
        w = np.zeros((m, words(n)), dtype=np.uint64)
        assert self.lib.f2o_fixed_weight(ptr(w), m, n, weight, seed) == 0
        return w

    def gauss_pls(self, w, n):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        m = w.shape[0]
        p = np.zeros(m, dtype=np.uint64)
        q = np.zeros(n, dtype=np.uint64)
        r = self.lib.f2o_gauss_pls(ptr(w), m, n, ptr(p), ptr(q))
        return w, p, q, r

    def recursive_q(self, m, n, cutoff, pivcols):
        piv = np.ascontiguousarray(pivcols, dtype=np.uint64)
        q = np.zeros(n, dtype=np.uint64)
        self.lib.f2o_recursive_q(m, n, cutoff, piv.size, ptr(piv) if piv.size else None, ptr(q))
        return q

    def mul(self, a, s, b, n):
        m = a.shape[0]
        c = np.zeros((m, words(n)), dtype=np.uint64)
        self.lib.f2o_mul(ptr(np.ascontiguousarray(a)), m, s, ptr(np.ascontiguousarray(b)), n, ptr(c))
        return c

    def pls_check(self, orig, packed, n, rank, p, q):
        m = orig.shape[0]
        return bool(self.lib.f2o_pls_check(ptr(np.ascontiguousarray(orig)), ptr(np.ascontiguousarray(packed)),
                                           m, n, rank, ptr(np.ascontiguousarray(p, dtype=np.uint64)),
                                           ptr(np.ascontiguousarray(q, dtype=np.uint64))))

    def digest(self, w):
        w = np.ascontiguousarray(w)
        return int(self.lib.f2o_digest(ptr(w), w.size))

    def gauss_rref(self, w, n):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        r = self.lib.f2o_gauss_rref(ptr(w), w.shape[0], n)
        return w, int(r)

    def m4ri_rref(self, w, n, k=0, full=True):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        r = self.lib.f2o_m4ri_rref(ptr(w), w.shape[0], n, k, int(full))
        if r < 0:
            raise ValueError("m4ri_rref: k must be in 0..8")
        return w, int(r)

    def rref_from_pls(self, w, n, rank, q):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        q = np.ascontiguousarray(q, dtype=np.uint64)
        if self.lib.f2o_rref_from_pls(ptr(w), w.shape[0], n, rank, ptr(q) if q.size else None, q.size):
            raise ValueError("rref_from_pls: invalid_argument")
        return w


class RefLib:
    """The reference library itself (built from /root/reference sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_randomize.argtypes = [u64p, sz, sz, C.c_double, C.c_uint64]
        L.ref_mmpf_pls.argtypes = [u64p, sz, sz, C.c_uint, u64p, u64p, u64p]
        L.ref_pls_recursive.argtypes = [u64p, sz, sz, C.c_uint, C.c_uint64, u64p, u64p, u64p]
        L.ref_gauss_pls.argtypes = [u64p, sz, sz, u64p, u64p, u64p]
        L.ref_rref_from_pls.argtypes = [u64p, sz, sz, C.c_uint64, u64p, sz]
        L.ref_gauss_rref.argtypes = [u64p, sz, sz, u64p]
        L.ref_m4ri_rref.argtypes = [u64p, sz, sz, C.c_uint, C.c_int, u64p]
        L.ref_hybrid_rref.argtypes = [u64p, sz, sz, C.c_uint, C.c_uint64, C.c_double, u64p]
        L.ref_rank.argtypes = [u64p, sz, sz, C.c_int, C.c_uint, C.c_uint64, C.c_double, u64p]
        L.ref_mul_m4rm.argtypes = [u64p, sz, sz, u64p, sz, C.c_uint, u64p]
        L.ref_mul_naive.argtypes = [u64p, sz, sz, u64p, sz, u64p]
        L.ref_trsm_lower_left_unit.argtypes = [u64p, sz, u64p, sz]
        L.ref_trsm_upper_left_unit.argtypes = [u64p, sz, u64p, sz]
        L.ref_default_cutoff_bytes.restype = sz
        L.ref_apply_rows.argtypes = [u64p, sz, sz, u64p, sz, C.c_int]
        L.ref_compress_columns.argtypes = [u64p, sz, sz, sz, u64p, sz]
        L.ref_auto_table_bits.argtypes = [sz]
        L.ref_auto_table_bits.restype = C.c_uint

    def randomize(self, m, n, density, seed):
        w = np.zeros((m, words(n)), dtype=np.uint64)
        assert self.lib.ref_randomize(ptr(w), m, n, density, seed) == 0
        return w

    def apply_rows(self, w, n, v, inverse=False):
        """Permutation::apply_rows[_inverse] (perm.cpp:25-38); returns (status, rows)."""
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        v = np.ascontiguousarray(v, dtype=np.uint64)
        rc = self.lib.ref_apply_rows(ptr(w), w.shape[0], n, ptr(v) if v.size else None, v.size, int(inverse))
        return rc, w

    def compress_columns(self, w, n, rank, q):
        """compress_columns(BitMatrix&, rank, Permutation) (perm.cpp:55-60); returns (status, matrix)."""
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        q = np.ascontiguousarray(q, dtype=np.uint64)
        rc = self.lib.ref_compress_columns(ptr(w), w.shape[0], n, rank, ptr(q) if q.size else None, q.size)
        return rc, w

    def _pls(self, fn, w, n, *extra):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        m = w.shape[0]
        p = np.zeros(m, dtype=np.uint64)
        q = np.zeros(n, dtype=np.uint64)
        r = np.zeros(1, dtype=np.uint64)
        rc = fn(ptr(w), m, n, *extra, ptr(p), ptr(q), ptr(r))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return w, p, q, int(r[0])

    def mmpf_pls(self, w, n, k=0):
        return self._pls(self.lib.ref_mmpf_pls, w, n, k)

    def pls_recursive(self, w, n, cutoff, k=0):
        return self._pls(self.lib.ref_pls_recursive, w, n, k, cutoff)

    def gauss_pls(self, w, n):
        return self._pls(self.lib.ref_gauss_pls, w, n)

    def gauss_rref(self, w, n):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        r = np.zeros(1, dtype=np.uint64)
        assert self.lib.ref_gauss_rref(ptr(w), w.shape[0], n, ptr(r)) == 0
        return w, int(r[0])

    def rref_from_pls(self, w, n, rank, q):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        q = np.ascontiguousarray(q, dtype=np.uint64)
        rc = self.lib.ref_rref_from_pls(ptr(w), w.shape[0], n, rank, ptr(q) if q.size else None, q.size)
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return w

    def m4ri_rref(self, w, n, k=0, full=True):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        r = np.zeros(1, dtype=np.uint64)
        rc = self.lib.ref_m4ri_rref(ptr(w), w.shape[0], n, k, int(full), ptr(r))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return w, int(r[0])

    def hybrid_rref(self, w, n, k=0, cutoff=0, threshold=0.15):
        w = np.array(w, dtype=np.uint64, copy=True, order="C")
        r = np.zeros(1, dtype=np.uint64)
        rc = self.lib.ref_hybrid_rref(ptr(w), w.shape[0], n, k, cutoff, threshold, ptr(r))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return w, int(r[0])

    def rank(self, w, n, algorithm=3, k=0, cutoff=0, threshold=0.15):
        w = np.ascontiguousarray(w, dtype=np.uint64)
        r = np.zeros(1, dtype=np.uint64)
        rc = self.lib.ref_rank(ptr(w), w.shape[0], n, algorithm, k, cutoff, threshold, ptr(r))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return int(r[0])

    def mul_m4rm(self, a, s, b, n, k=0):
        m = a.shape[0]
        c = np.zeros((m, words(n)), dtype=np.uint64)
        assert self.lib.ref_mul_m4rm(ptr(np.ascontiguousarray(a)), m, s, ptr(np.ascontiguousarray(b)), n, k, ptr(c)) == 0
        return c
