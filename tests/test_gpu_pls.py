"""GPU parity: the CUDA PLS engine through the C ABI vs the CPU oracle and the
reference's golden outputs.  Bit-exact: packed L/S, P, Q (tail included for the
recursive entry point), rank."""
import os

import numpy as np
import pytest

from oracle_lib import digest, words

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def upload(f2, w, n):
    return f2.DeviceMatrix.from_host(np.ascontiguousarray(w), n)


def check_against_oracle(f2, oracle, a, n, panel_bits=None, recursive_cutoff=None):
    m = a.shape[0]
    if panel_bits:
        f2.set_panel_bits(panel_bits)
    d = upload(f2, a, n)
    if recursive_cutoff is None:
        res = f2.mmpf_pls(d)
    else:
        res = f2.pls_recursive(d, f2.EliminationConfig(cutoff_bytes=recursive_cutoff))
    got = d.download()
    w, p, q, r = oracle.gauss_pls(a, n)
    assert res.rank == r
    assert (res.P == p).all(), "P differs"
    if recursive_cutoff is None:
        assert (res.Q == q).all(), "Q differs"
    else:
        assert (res.Q == oracle.recursive_q(m, n, recursive_cutoff, q[:r])).all(), "recursive Q differs"
    assert (got == w).all(), "packed L/S differs"
    if panel_bits:
        f2.set_panel_bits(1024)


@pytest.fixture(scope="module")
def small_cases():
    z = np.load(os.path.join(HERE, "golden", "small_cases.npz"))
    return [{k.split("_", 1)[1]: z[k] for k in z.files if k.startswith(f"{i}_")} for i in range(int(z["count"]))]


def test_randomize_bit_exact(f2, oracle):
    for (m, n, d, s) in [(1, 1, 0.5, 1), (3, 64, 0.5, 2), (17, 130, 0.3, 3), (64, 1000, 0.02, 4), (5, 70, 1.0, 5),
                         (5, 70, 0.0, 6), (257, 4097, 0.5, 7)]:
        a = f2.DeviceMatrix(m, n)
        a.randomize(d, s)
        assert (a.download() == oracle.randomize(m, n, d, s)).all(), (m, n, d)
        assert a.digest() == digest(oracle.randomize(m, n, d, s))


def test_golden_small_cases_mmpf_and_recursive(f2, small_cases):
    """Reference outputs (mmpf_pls and pls_recursive at the case's cutoff)."""
    for c in small_cases:
        n = int(c["n"])
        d = upload(f2, c["a"], n)
        res = f2.mmpf_pls(d)
        assert res.rank == int(c["mm_r"])
        assert (d.download() == c["mm_w"]).all() and (res.P == c["mm_p"]).all() and (res.Q == c["mm_q"]).all()
        d = upload(f2, c["a"], n)
        res = f2.pls_recursive(d, f2.EliminationConfig(cutoff_bytes=int(c["cutoff"])))
        assert res.rank == int(c["rc_r"])
        assert (d.download() == c["rc_w"]).all() and (res.P == c["rc_p"]).all() and (res.Q == c["rc_q"]).all()


@pytest.mark.parametrize("panel", [64, 128, 512, 1024])
def test_random_shapes_all_panels(f2, oracle, panel):
    rng = np.random.default_rng(panel)
    for t in range(25):
        m, n = int(rng.integers(1, 700)), int(rng.integers(1, 700))
        d = [0.01, 0.05, 0.3, 0.5, 0.9][t % 5]
        a = oracle.randomize(m, n, d, int(rng.integers(1, 2 ** 62)))
        check_against_oracle(f2, oracle, a, n, panel_bits=panel, recursive_cutoff=[8, 4096, 1 << 20][t % 3])


def test_rank_deficient_and_structured(f2, oracle):
    rng = np.random.default_rng(5)
    cases = []
    # X*Y rank-deficient (config-4 shape, scaled down)
    x = oracle.randomize(600, 300, 0.5, 1)
    y = oracle.randomize(300, 600, 0.5, 2)
    cases.append((oracle.mul(x, 300, y, 600), 600))
    # fixed weight sparse (config-5 shape, scaled down)
    cases.append((oracle.fixed_weight(256, 2048, 8, 3), 2048))
    cases.append((oracle.fixed_weight(300, 300, 2, 4), 300))
    # duplicate rows, zero columns, identity, all-ones
    a = oracle.randomize(200, 190, 0.5, 6)
    a[100:] = a[:100]
    a[:, 1] = 0
    cases.append((a, 190))
    idm = np.zeros((300, words(300)), np.uint64)
    for i in range(300):
        idm[i, i // 64] |= np.uint64(1) << np.uint64(i % 64)
    cases.append((idm, 300))
    cases.append((oracle.randomize(70, 70, 1.0, 1), 70))
    cases.append((np.zeros((100, words(130)), np.uint64), 130))
    for a, n in cases:
        for panel in (64, 1024):
            check_against_oracle(f2, oracle, a, n, panel_bits=panel)
            check_against_oracle(f2, oracle, a, n, panel_bits=panel, recursive_cutoff=2048)


def test_tall_and_wide_multiword(f2, oracle):
    for (m, n, d) in [(3000, 100, 0.5), (100, 3000, 0.5), (2000, 2000, 0.02), (1500, 1500, 0.5), (130, 4100, 0.1)]:
        a = oracle.randomize(m, n, d, m * 7 + n)
        check_against_oracle(f2, oracle, a, n)
        check_against_oracle(f2, oracle, a, n, recursive_cutoff=1 << 16)


def test_worked_examples(f2):
    # test_mmpf.cpp:140-155 and test_gauss.cpp:45-53
    w = np.array([[0b11], [0b01]], np.uint64)  # rows "11", "10" (col 0 = LSB)
    d = upload(f2, w, 2)
    r = f2.mmpf_pls(d)
    assert r.rank == 2 and list(r.P) == [0, 1] and list(r.Q) == [0, 1]
    assert (d.download() == np.array([[0b11], [0b11]], np.uint64)).all()
    w = np.array([[0b10], [0b01]], np.uint64)  # "01", "10"
    d = upload(f2, w, 2)
    r = f2.mmpf_pls(d)
    assert list(r.P) == [1, 1] and (d.download() == np.array([[0b01], [0b10]], np.uint64)).all()


def test_empty_and_errors(f2):
    import ctypes as C
    d = f2.DeviceMatrix(0, 5)
    r = f2.mmpf_pls(d)
    assert r.rank == 0 and list(r.Q) == list(range(5))
    d = f2.DeviceMatrix(5, 0)
    assert f2.pls_recursive(d).rank == 0
    d = f2.DeviceMatrix(4, 4)
    with pytest.raises(ValueError):
        f2.mmpf_pls(d, k=9)  # mmpf.cpp:90
    with pytest.raises(IndexError):
        d.window(0, 0, 5, 4)
    L = f2.load_library()
    p = np.zeros(3, np.uint64)
    q = np.zeros(4, np.uint64)
    rank = C.c_uint64()
    rc = L.f2_mmpf_pls(d.handle, f2.Window(0, 0, 4, 4).c(), p.ctypes.data_as(C.POINTER(C.c_uint64)), 3,
                       q.ctypes.data_as(C.POINTER(C.c_uint64)), 4, 0, C.byref(rank))
    assert rc == f2.F2_INVALID_ARGUMENT  # mmpf.cpp:85-86
    rc = L.f2_mmpf_pls(d.handle, f2.Window(0, 0, 5, 4).c(), p.ctypes.data_as(C.POINTER(C.c_uint64)), 5,
                       q.ctypes.data_as(C.POINTER(C.c_uint64)), 4, 0, C.byref(rank))
    assert rc == f2.F2_OUT_OF_RANGE
    with pytest.raises(ValueError):
        f2.pls_recursive(d, f2.EliminationConfig(hybrid_threshold=1.5))  # pls.cpp:57-61


def test_windows(f2, oracle):
    """MatrixWindow entry points touch only the window (bitmat.hpp:237-238)."""
    rng = np.random.default_rng(3)
    for t in range(12):
        M, N = 300, 400
        big = oracle.randomize(M, N, 0.5, 100 + t)
        r0, r1 = sorted(int(x) for x in rng.integers(0, M, 2))
        c0, c1 = sorted(int(x) for x in rng.integers(0, N, 2))
        r1, c1 = r1 + 1, c1 + 1
        d = upload(f2, big, N)
        win = d.window(r0, c0, r1, c1)
        res = f2.mmpf_pls(d, window=win) if t % 2 else f2.pls_recursive(d, f2.EliminationConfig(cutoff_bytes=256),
                                                                      window=win)
        got = d.download()
        # extract the window with numpy (bit by bit) and run the oracle on it
        bits = np.unpackbits(big.view(np.uint8), axis=1, bitorder="little")[:, :N]
        sub = bits[r0:r1, c0:c1]
        n = c1 - c0
        subw = np.zeros((r1 - r0, words(n)), np.uint64)
        pb = np.packbits(np.pad(sub, ((0, 0), (0, words(n) * 64 - n))), axis=1, bitorder="little")
        subw[:] = pb.view(np.uint64)
        w, p, q, r = oracle.gauss_pls(subw, n)
        gb = np.unpackbits(got.view(np.uint8), axis=1, bitorder="little")[:, :N]
        wb = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")[:, :n]
        assert res.rank == r and (res.P == p).all()
        assert (gb[r0:r1, c0:c1] == wb).all()
        outside = bits.copy()
        outside[r0:r1, c0:c1] = gb[r0:r1, c0:c1]
        assert (gb == outside).all(), "bits outside the window changed"


@pytest.mark.parametrize("pinned", [True, False])
def test_host_entry_points_streamed_download(f2, oracle, pinned):
    """f2_*_host: upload, decompose, download.  With a pinned buffer the finished
    pivot rows stream back during the factorisation (valid while every panel is
    full rank, redone otherwise): full-rank, rank-deficient, tall and wide inputs."""
    cases = [(3000, 3000, 0.5, None), (2500, 2600, 0.5, 300), (4100, 1500, 0.5, None), (1200, 5000, 0.5, None),
             (2048, 2048, 0.02, None)]
    for (m, n, d, inner) in cases:
        if inner:
            x = oracle.randomize(m, inner, 0.5, 5)
            y = oracle.randomize(inner, n, 0.5, 6)
            a = oracle.mul(x, inner, y, n)
        else:
            a = oracle.randomize(m, n, d, m + n)
        w, p, q, r = oracle.gauss_pls(a, n)
        for recursive in (True, False):
            h = f2.pinned_empty(a.shape) if pinned else np.empty_like(a)
            np.copyto(h, a)
            if recursive:
                res = f2.pls_recursive_host(h, n, f2.EliminationConfig(cutoff_bytes=4096))
                qq = oracle.recursive_q(m, n, 4096, q[:r])
            else:
                res = f2.mmpf_pls_host(h, n)
                qq = q
            assert res.rank == r and (res.P == p).all() and (res.Q == qq).all(), (m, n, recursive)
            assert (h == w).all(), (m, n, recursive, "packed")


@pytest.mark.parametrize("m,n,kind", [(4096, 16384, "dense"), (5000, 16384, "xy"), (3500, 16448, "sparse"),
                                      (12288, 32768, "dense"), (10000, 20480, "xy")])
def test_host_streamed_upload(f2, oracle, m, n, kind):
    """Pinned host buffers with >= 16 panels: the engine uploads the matrix itself in
    column groups and factors the first panels while the rest is in flight (api.cu,
    upload_plan).  Small cases against the Gaussian oracle, large ones against the same
    decomposition of a device matrix (no streamed upload), which the oracle pins elsewhere."""
    if kind == "xy":
        inner = m // 2
        a = oracle.mul(oracle.randomize(m, inner, 0.5, 5), inner, oracle.randomize(inner, n, 0.5, 6), n)
    elif kind == "sparse":
        a = oracle.fixed_weight(m, n, 4, 7)
    else:
        a = oracle.randomize(m, n, 0.5, m + n)
    cfg = f2.EliminationConfig(cutoff_bytes=4096)
    if m * n <= 5000 * 16448:
        w, p, q, r = oracle.gauss_pls(a, n)
        qr = oracle.recursive_q(m, n, 4096, q[:r])
    else:
        d = f2.DeviceMatrix.from_host(a, n)
        res = f2.pls_recursive(d, cfg)
        w, p, qr, r = d.download(), res.P, res.Q, res.rank
        d2 = f2.DeviceMatrix.from_host(a, n)
        q = f2.mmpf_pls(d2).Q
    for recursive in (True, False):
        for rep in range(2):  # the second call replays the cached graph
            h = f2.pinned_empty(a.shape)
            np.copyto(h, a)
            res = f2.pls_recursive_host(h, n, cfg) if recursive else f2.mmpf_pls_host(h, n)
            assert res.rank == r and (res.P == p).all(), (m, n, kind, recursive, rep)
            assert (res.Q == (qr if recursive else q)).all(), (m, n, kind, recursive, rep, "Q")
            assert (h == w).all(), (m, n, kind, recursive, rep, "packed")


def test_pivot_search_window_tiers(f2, oracle):
    """The fast pivot search looks at the first 96 window slots, then all 128, then falls back
    to the general search (csrc/leaf_body.cuh row_pivots, panel.cu): inputs whose pivots sit
    only in slots 96-127, only past the window, or alternate between the tiers from leaf to
    leaf, with zero columns in between (gauss.cpp:33-49 is the rule in every tier)."""
    rng = np.random.default_rng(96128)
    cases = []
    for m, n, zero_rows in [(200, 64, 96), (200, 200, 100), (300, 130, 127), (300, 200, 128), (400, 256, 200),
                            (130, 64, 97), (97, 97, 96), (129, 300, 128), (1000, 192, 96)]:
        a = oracle.randomize(m, n, 0.5, int(rng.integers(1, 2 ** 62)))
        a[:zero_rows, :] = 0
        cases.append((a, n))
    # per 64-column leaf a different band of rows is nonzero: 0-95, 96-127, past 128, none
    m, n = 520, 512
    a = np.zeros((m, words(n)), dtype=np.uint64)
    full = oracle.randomize(m, n, 0.5, 7)
    bands = [(0, 96), (96, 128), (128, 520), (0, 0), (100, 120), (300, 310), (0, 520), (127, 129)]
    for j, (r0, r1) in enumerate(bands):
        a[r0:r1, j] = full[r0:r1, j]
    cases.append((a, n))
    # sparse columns: few candidates, most of them deep in the order
    a = np.zeros((700, words(256)), dtype=np.uint64)
    for c in range(256):
        for r in rng.integers(0, 700, size=2):
            a[r, c // 64] |= np.uint64(1) << np.uint64(c % 64)
    cases.append((a, 256))
    for a, n in cases:
        check_against_oracle(f2, oracle, a, n, recursive_cutoff=4096)
        check_against_oracle(f2, oracle, a, n)


def test_graph_cache_across_buffers_and_shapes(f2, oracle):
    """The engine replays cached CUDA graphs keyed by matrix buffer and shape (csrc/api.cu,
    run_engine): six live buffers over four cache slots, two shapes interleaved, different
    contents per buffer -- every call must factor its own matrix (a stale buffer pointer in a
    replayed or in-place updated graph would factor another one)."""
    shapes = [(2048, 2048), (2304, 2176)]
    mats = []
    for i in range(6):
        m, n = shapes[i % 2]
        a = oracle.randomize(m, n, 0.5, 9000 + i)
        mats.append((a, m, n, oracle.gauss_pls(a, n)))
    bufs = [f2.DeviceMatrix(m, n) for (_, m, n, _) in mats]
    for rnd in range(3):
        for i in ([0, 1, 2, 3, 4, 5] if rnd != 1 else [5, 3, 1, 4, 2, 0]):
            a, m, n, (w, p, q, r) = mats[i]
            bufs[i].copy_from(upload(f2, a, n))
            res = f2.pls_recursive(bufs[i], f2.EliminationConfig(cutoff_bytes=1 << 16))
            assert res.rank == r and (res.P == p).all(), (rnd, i)
            assert (bufs[i].download() == w).all(), (rnd, i)
            assert (res.Q == oracle.recursive_q(m, n, 1 << 16, q[:r])).all(), (rnd, i)
