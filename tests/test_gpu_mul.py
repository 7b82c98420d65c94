"""GPU: the standalone multiply / TRSM entry points (mul.hpp:17-28) against the CPU
oracle.  Shapes cover both GEMM paths of the engine: the SMEM table kernel (K < 256
or thin products) and the tensor-core kernel (K >= 256, >= 128 rows, >= 256 columns;
K > 1024 runs in 1024-bit chunks), windows at word and bit offsets, and the
reference's error conditions (mul.cpp:103-111)."""
import numpy as np
import pytest

from oracle_lib import words

pytestmark = pytest.mark.gpu


def rand_words(rng, m, n):
    w = rng.integers(0, 1 << 63, size=(m, words(n)), dtype=np.uint64) ^ \
        (rng.integers(0, 2, size=(m, words(n)), dtype=np.uint64) << np.uint64(63))
    if n % 64:
        w[:, -1] &= np.uint64((1 << (n % 64)) - 1)
    return w


def get_bits(w, r0, r1, c0, c1):
    """rows [r0, r1), columns [c0, c1) of a packed matrix, re-packed from column 0."""
    m, n = r1 - r0, c1 - c0
    cols = np.arange(c0, c1)
    bits = (w[r0:r1, cols // 64] >> (cols % 64).astype(np.uint64)) & np.uint64(1)
    out = np.zeros((m, words(n)), np.uint64)
    for j in range(n):
        out[:, j // 64] |= bits[:, j] << np.uint64(j % 64)
    return out


@pytest.mark.parametrize("p,s,q", [(100, 37, 70), (64, 200, 130), (300, 300, 500), (129, 256, 256),
                                   (1000, 1500, 700), (2048, 1024, 2048), (777, 2100, 1300)])
def test_addmul_vs_oracle(f2, oracle, p, s, q):
    rng = np.random.default_rng(p * 7 + s * 13 + q)
    a, b, c = rand_words(rng, p, s), rand_words(rng, s, q), rand_words(rng, p, q)
    dc = f2.DeviceMatrix.from_host(c, q)
    f2.addmul(dc, f2.DeviceMatrix.from_host(a, s), f2.DeviceMatrix.from_host(b, q))
    assert (dc.download() == (c ^ oracle.mul(a, s, b, q))).all()


def test_mul_m4rm_vs_reference(f2, oracle):
    rng = np.random.default_rng(5)
    for m, s, n in [(513, 1024, 900), (4096, 3000, 2500), (10, 10, 10)]:
        a, b = rand_words(rng, m, s), rand_words(rng, s, n)
        got = f2.mul_m4rm(f2.DeviceMatrix.from_host(a, s), f2.DeviceMatrix.from_host(b, n)).download()
        assert (got == oracle.mul(a, s, b, n)).all(), (m, s, n)


@pytest.mark.parametrize("k", [1, 8, 9, 33, 36, 44, 45, 50, 60, 64])
def test_addmul_mmpf_streaming_kernel(f2, oracle, k):
    """K <= 64 takes the HBM-streaming MMPF table-apply: every table layout (1-4 8-bit tables
    at 4096- to 1024-bit tiles for K <= 32; 5-10 7-bit tables at 1024-bit tiles for K > 32),
    a C window starting at an odd word (tile-edge lanes with one valid word), rows across
    2048-row blocks (K <= 32) and 8192-row blocks (K = 64)."""
    rng = np.random.default_rng(k)
    p, q, c0 = 9000 if k == 64 else 4500, 5000, 64 * 3
    a, b = rand_words(rng, p, k), rand_words(rng, k, q)
    big = rand_words(rng, p, q + c0 + 64)
    dc = f2.DeviceMatrix.from_host(big, q + c0 + 64)
    f2.addmul(dc, f2.DeviceMatrix.from_host(a, k), f2.DeviceMatrix.from_host(b, q), wc=dc.window(0, c0, p, c0 + q))
    got = dc.download()
    exp = big.copy()
    prod = oracle.mul(a, k, b, q)
    exp[:, c0 // 64:c0 // 64 + words(q)] ^= prod
    assert (got == exp).all()


@pytest.mark.parametrize("c0", [64, 69])
def test_addmul_windows(f2, oracle, c0):
    """C, A, B as windows of larger matrices: only the C window changes."""
    rng = np.random.default_rng(c0)
    p, s, q = 600, 700, 520
    big_c = rand_words(rng, p + 50, q + c0 + 90)
    big_a = rand_words(rng, p + 20, s + 130)
    big_b = rand_words(rng, s + 10, q + 64)
    dc = f2.DeviceMatrix.from_host(big_c, q + c0 + 90)
    da = f2.DeviceMatrix.from_host(big_a, s + 130)
    db = f2.DeviceMatrix.from_host(big_b, q + 64)
    f2.addmul(dc, da, db, wc=dc.window(30, c0, 30 + p, c0 + q), wa=da.window(7, 65, 7 + p, 65 + s),
              wb=db.window(3, 64, 3 + s, 64 + q))
    prod = oracle.mul(get_bits(big_a, 7, 7 + p, 65, 65 + s), s, get_bits(big_b, 3, 3 + s, 64, 64 + q), q)
    got = dc.download()
    n_c = q + c0 + 90
    exp = big_c.copy()
    cols = np.arange(q)
    pbits = (prod[:, cols // 64] >> (cols % 64).astype(np.uint64)) & np.uint64(1)
    for j in range(q):
        col = c0 + j
        exp[30:30 + p, col // 64] ^= pbits[:, j] << np.uint64(col % 64)
    assert (got == exp).all()
    assert n_c == dc.ncols


@pytest.mark.parametrize("r,nb", [(60, 100), (700, 900), (2500, 1100)])
def test_trsm_lower_left_unit(f2, oracle, r, nb):
    """B <- L^{-1} B: L * B' == B with L's unit lower part (upper part ignored)."""
    rng = np.random.default_rng(r)
    lw, b = rand_words(rng, r, r), rand_words(rng, r, nb)
    dl, db = f2.DeviceMatrix.from_host(lw, r), f2.DeviceMatrix.from_host(b, nb)
    f2.trsm_lower_left_unit(dl, db)
    x = db.download()
    unit = lw.copy()
    for i in range(r):  # keep the strictly lower part, put 1 on the diagonal
        w, bit = divmod(i, 64)
        unit[i, w] &= np.uint64((1 << bit) - 1)
        unit[i, w + 1:] = 0
        unit[i, w] |= np.uint64(1 << bit)
    assert (oracle.mul(unit, r, x, nb) == b).all()
    assert (dl.download() == lw).all()


@pytest.mark.parametrize("r,nb", [(2, 5), (64, 100), (700, 900), (2500, 1100)])
def test_trsm_upper_left_unit(f2, oracle, r, nb):
    """B <- U^{-1} B (mul.cpp:133-155): U * B' == B with U's unit upper part (lower ignored),
    and a window case at bit offsets."""
    rng = np.random.default_rng(r + 1)
    uw, b = rand_words(rng, r, r), rand_words(rng, r, nb)
    du, db = f2.DeviceMatrix.from_host(uw, r), f2.DeviceMatrix.from_host(b, nb)
    f2.trsm_upper_left_unit(du, db)
    x = db.download()
    unit = uw.copy()
    for i in range(r):  # keep the strictly upper part, put 1 on the diagonal
        w, bit = divmod(i, 64)
        unit[i, :w] = 0
        unit[i, w] &= ~np.uint64((1 << (bit + 1)) - 1) if bit < 63 else np.uint64(0)
        unit[i, w] |= np.uint64(1 << bit)
    assert (oracle.mul(unit, r, x, nb) == b).all()
    assert (du.download() == uw).all()


def test_trsm_upper_window(f2, oracle):
    rng = np.random.default_rng(9)
    r, nb = 300, 200
    bigu = rand_words(rng, r + 10, r + 77)
    bigb = rand_words(rng, r + 5, nb + 70)
    du, db = f2.DeviceMatrix.from_host(bigu, r + 77), f2.DeviceMatrix.from_host(bigb, nb + 70)
    f2.trsm_upper_left_unit(du, db, wu=du.window(3, 70, 3 + r, 70 + r), wb=db.window(2, 5, 2 + r, 5 + nb))
    got = db.download()
    u = get_bits(bigu, 3, 3 + r, 70, 70 + r)
    for i in range(r):
        w, bit = divmod(i, 64)
        u[i, :w] = 0
        u[i, w] &= ~np.uint64((1 << (bit + 1)) - 1) if bit < 63 else np.uint64(0)
        u[i, w] |= np.uint64(1 << bit)
    x = get_bits(got, 2, 2 + r, 5, 5 + nb)
    assert (oracle.mul(u, r, x, nb) == get_bits(bigb, 2, 2 + r, 5, 5 + nb)).all()
    outside = got.copy()
    ref = bigb.copy()
    for i in range(2, 2 + r):  # bits outside the window untouched
        for j in range(5, 5 + nb):
            wd, bt = divmod(j, 64)
            m = np.uint64(1) << np.uint64(bt)
            outside[i, wd] &= ~m
            ref[i, wd] &= ~m
    assert (outside == ref).all()


def test_mul_errors(f2):
    """invalid_argument (mul.cpp:103-111) surfaces as ValueError."""
    a, b = f2.DeviceMatrix(10, 20), f2.DeviceMatrix(21, 5)
    with pytest.raises(ValueError):
        f2.mul_m4rm(a, b)
    c = f2.DeviceMatrix(10, 5)
    with pytest.raises(ValueError):
        f2.addmul(c, a, b)
    sq = f2.DeviceMatrix(300, 300)
    with pytest.raises(ValueError):  # C aliases A
        f2.addmul(sq, sq, f2.DeviceMatrix(300, 300))
    with pytest.raises(ValueError):
        f2.trsm_lower_left_unit(f2.DeviceMatrix(10, 11), f2.DeviceMatrix(10, 4))
