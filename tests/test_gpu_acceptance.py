"""GPU: the reference's acceptance criteria (tests/acceptance.cpp) on the engine —
RREF agreement across the algorithms (:64-100), reconstruction P^-1 L S = A on every
decomposition path (:102-134), rank sensitivity on matrices of known rank (:136-157)
and cutoff invariance of rank + RREF (:189-223).  120 / 60 random matrices instead of the
reference's 520 / 320, so the suite stays in seconds; every output is checked against the
CPU oracle bit for bit."""
import numpy as np
import pytest

from oracle_lib import words

pytestmark = pytest.mark.gpu


def shapes(rng, count, lo=1, hi=700):
    for t in range(count):
        yield int(rng.integers(lo, hi)), int(rng.integers(lo, hi)), [0.5, 0.1, 0.02, 0.9][t % 4]


def test_rref_agreement_across_algorithms(f2, oracle):
    """acceptance.cpp:64-100: gauss / m4ri / pls / hybrid give the same RREF and rank."""
    rng = np.random.default_rng(64)
    for m, n, dens in shapes(rng, 120):
        a = oracle.randomize(m, n, dens, int(rng.integers(1 << 40)))
        want, wr = oracle.gauss_rref(a, n)
        outs = []
        d = f2.DeviceMatrix.from_host(a, n)
        outs.append((f2.rref(d, f2.EliminationConfig(cutoff_bytes=4096)), d.download()))
        d = f2.DeviceMatrix.from_host(a, n)
        outs.append((f2.m4ri_rref(d, int(rng.integers(0, 9))), d.download()))
        d = f2.DeviceMatrix.from_host(a, n)
        outs.append((f2.hybrid_rref(d, f2.EliminationConfig(algorithm=f2.ALG_HYBRID)), d.download()))
        for r, got in outs:
            assert r == wr and (got == want).all(), (m, n, dens)


def test_reconstruction_on_every_path(f2, oracle):
    """acceptance.cpp:102-134: P^-1 (L S) == A for mmpf_pls and pls_recursive at several
    cutoffs, including rank-deficient products."""
    rng = np.random.default_rng(102)
    for t, (m, n, dens) in enumerate(shapes(rng, 60, 2, 900)):
        a = oracle.randomize(m, n, dens, 500 + t)
        if t % 3 == 0:  # rank deficient: a product through a thin inner dimension
            k = max(1, min(m, n) // 3)
            a = oracle.mul(oracle.randomize(m, k, 0.5, 7 + t), k, oracle.randomize(k, n, 0.5, 9 + t), n)
        runs = [("mmpf", lambda d: f2.mmpf_pls(d))]
        for cut in (8, 4096, 1 << 30):
            runs.append((f"pls{cut}", lambda d, c=cut: f2.pls_recursive(d, f2.EliminationConfig(cutoff_bytes=c))))
        for name, fn in runs:
            d = f2.DeviceMatrix.from_host(a, n)
            res = fn(d)
            assert oracle.pls_check(a, d.download(), n, res.rank, res.P, res.Q), (name, m, n)


def test_rank_sensitivity(f2, oracle):
    """acceptance.cpp:136-157: matrices of every prescribed rank r = X (n x r) * Y (r x n)."""
    rng = np.random.default_rng(136)
    n = 640
    for r in (0, 1, 2, 63, 64, 65, 320, 639, 640):
        if r == 0:
            a = np.zeros((n, words(n)), np.uint64)
        else:
            x = oracle.randomize(n, r, 0.5, int(rng.integers(1 << 40)))
            y = oracle.randomize(r, n, 0.5, int(rng.integers(1 << 40)))
            a = oracle.mul(x, r, y, n)
        want = oracle.gauss_rref(a, n)[1]
        assert want <= r
        d = f2.DeviceMatrix.from_host(a, n)
        for alg in range(5):
            assert f2.rank(d, f2.EliminationConfig(algorithm=alg)) == want


def test_cutoff_invariance(f2, oracle):
    """acceptance.cpp:189-223: rank, packed result, P and the RREF do not depend on the
    cutoff (512 x 512 and a wide 300 x 1500); Q agrees on its rank prefix and its tail
    follows the recursion replay."""
    for m, n, seed in ((512, 512, 1), (300, 1500, 2), (1500, 300, 3)):
        a = oracle.randomize(m, n, 0.5, seed)
        base = None
        for cut in (8, 512, 4096, 1 << 20, 1 << 30):
            d = f2.DeviceMatrix.from_host(a, n)
            res = f2.pls_recursive(d, f2.EliminationConfig(cutoff_bytes=cut))
            packed = d.download()
            assert (res.Q == oracle.recursive_q(m, n, cut, res.Q[:res.rank])).all()
            if base is None:
                base = (res.rank, packed, res.P, res.Q[:res.rank])
            else:
                assert res.rank == base[0] and (packed == base[1]).all() and (res.P == base[2]).all()
                assert (res.Q[:res.rank] == base[3]).all()
            f2.rref_from_pls(d, res.rank, res.Q[:res.rank])
            assert (d.download() == oracle.gauss_rref(a, n)[0]).all()
