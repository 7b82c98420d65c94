"""GPU: the standalone permutation entry points against the reference itself
(oracle/_ref: Permutation::apply_rows[_inverse] and compress_columns, perm.cpp:25-60)
and the C restatement: random transposition vectors, windows, compressions of real
PLS results and of arbitrary Q prefixes, and the reference's invalid_argument cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _transpositions(rng, m, length):
    """LAPACK-form vector: v[i] >= i (a valid Permutation, perm.hpp:36-40)."""
    return np.array([rng.integers(i, m) for i in range(length)], dtype=np.uint64)


@pytest.mark.parametrize("m,n,length", [(1, 1, 1), (64, 64, 64), (300, 70, 300), (1000, 513, 700), (4096, 2048, 4096),
                                        (777, 1, 10)])
@pytest.mark.parametrize("inverse", [False, True])
def test_apply_rows_vs_reference(f2, oracle, reflib, m, n, length, inverse):
    rng = np.random.default_rng(m * 7 + n + length)
    a = oracle.randomize(m, n, 0.5, m + n)
    v = _transpositions(rng, m, length)
    rc, want = reflib.apply_rows(a, n, v, inverse)
    assert rc == 0
    d = f2.DeviceMatrix.from_host(a, n)
    f2.apply_rows(d, v, inverse=inverse)
    assert (d.download() == want).all()


def test_apply_rows_round_trip_and_window(f2, oracle):
    """apply_rows_inverse undoes apply_rows (test_perm.cpp:37-47); on a window the rows and
    columns outside stay untouched."""
    rng = np.random.default_rng(5)
    m, n = 900, 1000
    a = oracle.randomize(m, n, 0.5, 17)
    d = f2.DeviceMatrix.from_host(a, n)
    v = _transpositions(rng, m, m)
    f2.apply_rows(d, v)
    f2.apply_rows(d, v, inverse=True)
    assert (d.download() == a).all()
    w = d.window(100, 37, 700, 901)
    vw = _transpositions(rng, 600, 600)
    f2.apply_rows(d, vw, window=w)
    got = d.download()
    # the same swaps on a host copy, bit by bit inside the window only
    ref = a.copy()
    bits = np.unpackbits(ref.view(np.uint8), axis=1, bitorder="little")[:, :n]
    sub = bits[100:700, 37:901]
    for i, j in enumerate(vw):
        j = int(j)
        if j != i:
            sub[[i, j]] = sub[[j, i]]
    bits[100:700, 37:901] = sub
    packed = np.packbits(np.pad(bits, ((0, 0), (0, ref.shape[1] * 64 - n))), axis=1, bitorder="little")
    assert (got == packed.view(np.uint64)).all()


@pytest.mark.parametrize("m,n,kind", [(200, 300, "xy"), (1000, 1000, "xy"), (512, 4096, "sparse"),
                                      (3000, 1500, "dense")])
def test_compress_columns_of_pls_results(f2, oracle, reflib, m, n, kind):
    """compress_columns on the uncompressed output of a PLS (L stored at the pivot
    columns) -- what the sharded path and the reference's mmpf driver (mmpf.cpp:112) do."""
    if kind == "xy":
        k = min(m, n) // 2
        a = oracle.mul(oracle.randomize(m, k, 0.5, 1), k, oracle.randomize(k, n, 0.5, 2), n)
    elif kind == "sparse":
        a = oracle.fixed_weight(m, n, 5, 3)
    else:
        a = oracle.randomize(m, n, 0.5, 4)
    w, p, q, r = oracle.gauss_pls(a, n)
    # undo the compression on the oracle's result: apply the swaps in reverse order
    unc = w.copy()
    bits = np.unpackbits(unc.view(np.uint8), axis=1, bitorder="little")[:, :n]
    for j in reversed(range(r)):
        qj = int(q[j])
        if qj != j:
            bits[j:, [j, qj]] = bits[j:, [qj, j]]
    unc = np.packbits(np.pad(bits, ((0, 0), (0, unc.shape[1] * 64 - n))), axis=1,
                      bitorder="little").view(np.uint64).copy()
    rc, want = reflib.compress_columns(unc, n, r, q)
    assert rc == 0 and (want == w).all()
    d = f2.DeviceMatrix.from_host(unc, n)
    f2.compress_columns(d, r, q)
    assert (d.download() == w).all()


@pytest.mark.parametrize("m,n,rank", [(64, 64, 10), (500, 800, 300), (2048, 300, 300)])
def test_compress_columns_arbitrary_q(f2, oracle, reflib, m, n, rank):
    """Any valid transposition prefix on arbitrary bits (not only PLS outputs)."""
    rng = np.random.default_rng(rank)
    a = oracle.randomize(m, n, 0.5, 99)
    q = _transpositions(rng, n, n)
    rc, want = reflib.compress_columns(a, n, rank, q)
    assert rc == 0
    d = f2.DeviceMatrix.from_host(a, n)
    f2.compress_columns(d, rank, q)
    assert (d.download() == want).all()


def test_perm_errors_match_reference(f2, oracle, reflib):
    """invalid_argument: rank > rows or > len(q) (perm.cpp:56-57); a permutation longer
    than the rows (perm.cpp:28, :35)."""
    a = oracle.randomize(10, 20, 0.5, 1)
    d = f2.DeviceMatrix.from_host(a, 20)
    q = np.arange(20, dtype=np.uint64)
    assert reflib.compress_columns(a, 20, 11, q)[0] == 1
    with pytest.raises(ValueError):
        f2.compress_columns(d, 11, q)
    assert reflib.compress_columns(a, 20, 5, q[:4])[0] == 1
    with pytest.raises(ValueError):
        f2.compress_columns(d, 5, q[:4])
    v = np.arange(11, dtype=np.uint64)
    for inverse in (False, True):
        assert reflib.apply_rows(a, 20, v, inverse)[0] == 1
        with pytest.raises(ValueError):
            f2.apply_rows(d, v, inverse=inverse)
    assert (d.download() == a).all()
