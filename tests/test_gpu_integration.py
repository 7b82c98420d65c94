"""GPU: the reference-side binding of INTEGRATION.md (integration/f2lin_gpu_adapter.hpp),
compiled against the reference's own headers and BitMatrix (oracle/Makefile target
`adapter`), decomposes reference BitMatrix objects through libf2gpu.so; the results
must equal the reference's pls_recursive / mmpf_pls (pls.hpp:44-45, mmpf.hpp:36) run on
the same matrices: packed L\\S, P, full Q (recursive tail included) and rank."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_lib import ROOT, ptr

pytestmark = pytest.mark.gpu
ADAPTER = os.path.join(ROOT, "oracle", "_ref", "libadapter.so")


@pytest.fixture(scope="module")
def adapter(f2):
    if not os.path.exists(ADAPTER):
        pytest.skip("oracle/_ref/libadapter.so not built (needs /root/reference at build time)")
    L = C.CDLL(ADAPTER)
    u64p = C.POINTER(C.c_uint64)
    L.adapter_pls.argtypes = [C.c_int, u64p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_uint, u64p, u64p, u64p]
    return L


def _run(adapter, recursive, a, m, n, cutoff=0, k=0):
    w = np.array(a, dtype=np.uint64, copy=True, order="C")
    p, q, r = np.zeros(m, np.uint64), np.zeros(n, np.uint64), np.zeros(1, np.uint64)
    rc = adapter.adapter_pls(int(recursive), ptr(w), m, n, cutoff, k, ptr(p), ptr(q), ptr(r))
    return rc, w, p, q, int(r[0])


@pytest.mark.parametrize("m,n,kind", [(1, 1, "dense"), (300, 500, "dense"), (2048, 2048, "dense"),
                                      (1500, 1500, "xy"), (700, 5000, "sparse"), (3000, 900, "dense")])
@pytest.mark.parametrize("recursive", [True, False])
def test_adapter_matches_reference(adapter, oracle, reflib, m, n, kind, recursive):
    if kind == "xy":
        a = oracle.mul(oracle.randomize(m, 400, 0.5, 1), 400, oracle.randomize(400, n, 0.5, 2), n)
    elif kind == "sparse":
        a = oracle.fixed_weight(m, n, 4, 3)
    else:
        a = reflib.randomize(m, n, 0.5, m + n)
    cutoff = 8192
    rc, w, p, q, r = _run(adapter, recursive, a, m, n, cutoff=cutoff)
    assert rc == 0
    want = reflib.pls_recursive(a, n, cutoff) if recursive else reflib.mmpf_pls(a, n)
    ww, wp, wq, wr = want
    assert r == wr and (p == wp).all() and (q == wq).all() and (w == ww).all()


def test_adapter_rethrows_like_reference(adapter, reflib):
    """k > 8 is invalid_argument in the reference (mmpf.cpp:90) and through the adapter."""
    a = reflib.randomize(64, 64, 0.5, 1)
    assert _run(adapter, False, a, 64, 64, k=9)[0] == 1
