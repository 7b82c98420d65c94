"""GPU parity for the echelonize entry points: rref_from_pls (pls.cpp:128-161) and
rref (PLS + rref_from_pls), bit-exact against the reference's outputs
(tests/golden) and the C restatement (oracle/f2oracle.c f2o_rref_from_pls,
f2o_gauss_rref)."""
import os

import numpy as np
import pytest

from oracle_lib import words

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def small_cases():
    z = np.load(os.path.join(HERE, "golden", "small_cases.npz"))
    return [{k.split("_", 1)[1]: z[k] for k in z.files if k.startswith(f"{i}_")} for i in range(int(z["count"]))]


def test_golden_rref_from_pls(f2, small_cases):
    for c in small_cases:
        n = int(c["n"])
        for w, r, q in [(c["rc_w"], int(c["rc_r"]), c["rc_q"]), (c["mm_w"], int(c["mm_r"]), c["mm_q"])]:
            d = f2.DeviceMatrix.from_host(np.ascontiguousarray(w), n)
            f2.rref_from_pls(d, r, q[:r])
            assert (d.download() == c["rref_w"]).all()
        d = f2.DeviceMatrix.from_host(np.ascontiguousarray(c["a"]), n)
        assert f2.rref(d, f2.EliminationConfig(cutoff_bytes=int(c["cutoff"]))) == int(c["rc_r"])
        assert (d.download() == c["rref_w"]).all()


def test_known_answers_and_errors(f2):
    # test_pls.cpp:115-135
    idm = np.array([[np.uint64(1) << np.uint64(i)] for i in range(8)], np.uint64)
    d = f2.DeviceMatrix.from_host(idm, 8)
    res = f2.pls_recursive(d)
    f2.rref_from_pls(d, res.rank, res.Q, p=res.P)
    assert (d.download() == idm).all()
    d = f2.DeviceMatrix.from_host(np.array([[3], [3]], np.uint64), 2)
    res = f2.pls_recursive(d)
    assert res.rank == 1
    f2.rref_from_pls(d, res.rank, res.Q, p=res.P)
    assert list(d.download()[:, 0]) == [3, 0]
    c = f2.DeviceMatrix.from_host(idm[:4].copy(), 4)
    with pytest.raises(ValueError):
        f2.rref_from_pls(c, 3, np.array([0, 3, 2, 3], np.uint64))
    with pytest.raises(ValueError):
        f2.rref_from_pls(c, 5, np.arange(4, dtype=np.uint64))
    with pytest.raises(ValueError):
        f2.rref_from_pls(c, 2, np.arange(1, dtype=np.uint64))       # Q shorter than rank
    with pytest.raises(ValueError):
        f2.rref_from_pls(c, 2, np.arange(4, dtype=np.uint64), p=np.arange(3, dtype=np.uint64))
    assert (c.download() == idm[:4]).all()
    f2.rref_from_pls(c, 0, np.zeros(0, np.uint64))                     # rank 0: everything cleared
    assert not c.download().any()


@pytest.mark.parametrize("shape", [(1, 1), (3, 200), (200, 3), (700, 900), (1500, 1100), (2100, 2100),
                                   (1100, 4000), (4000, 1300)])
def test_random_vs_oracle(f2, oracle, shape):
    m, n = shape
    rng = np.random.default_rng(m * 7919 + n)
    for d in [0.02, 0.5]:
        a = oracle.randomize(m, n, d, int(rng.integers(1, 2 ** 62)))
        want, wr = oracle.gauss_rref(a, n)
        dm = f2.DeviceMatrix.from_host(a, n)
        res = f2.pls_recursive(dm, f2.EliminationConfig(cutoff_bytes=4096))
        assert res.rank == wr
        packed = dm.download()
        f2.rref_from_pls(dm, res.rank, res.Q[:res.rank])
        got = dm.download()
        assert (got == want).all()
        assert (got == oracle.rref_from_pls(packed, n, res.rank, res.Q[:res.rank])).all()


def test_rank_deficient_products(f2, oracle):
    """X*Y with a narrow inner dimension (rank <= inner, Q far from identity)."""
    for (m, k, n) in [(1300, 300, 1700), (2500, 1030, 2600)]:
        x = oracle.randomize(m, k, 0.5, m + k)
        y = oracle.randomize(k, n, 0.5, k + n)
        a = oracle.mul(x, k, y, n)
        want, wr = oracle.gauss_rref(a, n)
        dm = f2.DeviceMatrix.from_host(a, n)
        assert f2.rref(dm) == wr
        assert (dm.download() == want).all()


def test_window(f2, oracle):
    """rref_from_pls on a window at unaligned offsets leaves the rest untouched."""
    M, N = 600, 700
    big = oracle.randomize(M, N, 0.5, 77)
    r0, c0, r1, c1 = 37, 93, 537, 613
    m, n = r1 - r0, c1 - c0
    sub = np.zeros((m, words(n)), np.uint64)
    for i in range(m):
        for j in range(n):
            if (int(big[r0 + i, (c0 + j) // 64]) >> ((c0 + j) % 64)) & 1:
                sub[i, j // 64] |= np.uint64(1) << np.uint64(j % 64)
    want, wr = oracle.gauss_rref(sub, n)
    d = f2.DeviceMatrix.from_host(big, N)
    w = d.window(r0, c0, r1, c1)
    assert f2.rref(d, window=w) == wr
    got = d.download()
    for i in range(M):
        for j in range(N):
            inside = r0 <= i < r1 and c0 <= j < c1
            b = (int(got[i, j // 64]) >> (j % 64)) & 1
            if inside:
                assert b == (int(want[i - r0, (j - c0) // 64]) >> ((j - c0) % 64)) & 1
            else:
                assert b == (int(big[i, j // 64]) >> (j % 64)) & 1


@pytest.mark.parametrize("m,n,dens,k", [(50, 70, 0.5, 0), (300, 200, 0.5, 3), (200, 900, 0.1, 8), (1500, 1300, 0.5, 0),
                                        (700, 700, 0.02, 1), (2100, 3000, 0.5, 5)])
def test_m4ri_rref_both_modes(f2, oracle, m, n, dens, k):
    """m4ri_rref (m4ri.cpp:68-87): full = the RREF; full=False = M4RI's block-reduced echelon
    form, bit for bit against the oracle's restatement (pinned to the reference in
    test_oracle.py)."""
    a = oracle.randomize(m, n, dens, m * 7 + n + k)
    if m > 10:
        a[m // 2] = a[3]  # rank deficient
    for full in (True, False):
        want, wr = oracle.m4ri_rref(a, n, k, full)
        d = f2.DeviceMatrix.from_host(a, n)
        assert f2.m4ri_rref(d, k, full) == wr
        assert (d.download() == want).all(), (m, n, k, full)


def test_m4ri_rref_vs_reference_and_errors(f2, oracle, reflib):
    a = reflib.randomize(600, 800, 0.3, 5)
    for full in (True, False):
        want, wr = reflib.m4ri_rref(a, 800, 0, full)
        d = f2.DeviceMatrix.from_host(a, 800)
        assert f2.m4ri_rref(d, 0, full) == wr and (d.download() == want).all()
    with pytest.raises(ValueError):
        f2.m4ri_rref(f2.DeviceMatrix(4, 4), 9)
    assert f2.m4ri_rref(f2.DeviceMatrix(0, 5), 9) == 0  # empty: returns before the k check


def test_hybrid_rref_and_rank(f2, oracle, reflib):
    rng = np.random.default_rng(3)
    for t, (m, n) in enumerate([(64, 64), (500, 700), (1200, 1000)]):
        a = reflib.randomize(m, n, [0.5, 0.05, 0.5][t], 10 + t)
        want, wr = reflib.hybrid_rref(a, n, 0, 4096, 0.15)
        d = f2.DeviceMatrix.from_host(a, n)
        assert f2.hybrid_rref(d, f2.EliminationConfig(cutoff_bytes=4096, algorithm=f2.ALG_HYBRID)) == wr
        assert (d.download() == want).all()
        d = f2.DeviceMatrix.from_host(a, n)
        for alg in range(5):
            assert f2.rank(d, f2.EliminationConfig(algorithm=alg)) == wr
        assert (d.download() == a).all()  # rank leaves A alone
    with pytest.raises(ValueError):
        f2.hybrid_rref(f2.DeviceMatrix(3, 3), f2.EliminationConfig(hybrid_threshold=1.5))
    with pytest.raises(ValueError):
        f2.rank(f2.DeviceMatrix(3, 3), f2.EliminationConfig(k=9, algorithm=f2.ALG_MMPF))
    assert f2.rank(f2.DeviceMatrix(3, 3), f2.EliminationConfig(k=9, algorithm=f2.ALG_GAUSS)) == 0
