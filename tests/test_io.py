"""CPU: the native BMF2/ASCII readers and writers (csrc/io.cu, host entry points)
against files written by the reference's io::write_matrix (tests/golden/io/), the
reference's own io unit tests (test_io.cpp, cited per case) and, when
oracle/_ref is built, live differential runs including mutated files."""
import ctypes as C
import os
import random

import numpy as np
import pytest

from oracle_lib import words

HERE = os.path.dirname(os.path.abspath(__file__))
IO = os.path.join(HERE, "golden", "io")


@pytest.fixture(scope="module")
def fio():
    import paper_1006_1744_b200 as f2
    from paper_1006_1744_b200 import io
    f2.load_library()
    return io


def golden_files():
    z = np.load(os.path.join(IO, "matrices.npz"))
    out = []
    for i in range(int(z["count"])):
        a, n = z[f"m{i}"], int(z[f"n{i}"])
        out.append((i, a, n))
    return out


def path_of(i, a, n, ext):
    return os.path.join(IO, f"mat{i}_{a.shape[0]}x{n}.{ext}")


def test_golden_read_and_write_bytes(fio, tmp_path):
    for i, a, n in golden_files():
        for ext, fmt in [("txt", fio.Format.ascii), ("bmf2", fio.Format.binary)]:
            p = path_of(i, a, n, ext)
            m2, n2, f = fio.probe(p)
            assert (m2, n2, f) == (a.shape[0], n, fmt)
            w, n3, f3 = fio.read_matrix_host(p)
            assert n3 == n and f3 == fmt and (w == a).all()
            out = tmp_path / f"o.{ext}"
            fio.write_matrix_host(out, a, n, fmt)
            assert out.read_bytes() == open(p, "rb").read()


def test_known_answers(fio, tmp_path):
    # test_io.cpp:12-21 ascii round trip
    a = np.array([[0b101], [0b010]], np.uint64)
    p = tmp_path / "a.txt"
    fio.write_matrix_host(p, a, 3, fio.Format.ascii)
    assert p.read_bytes() == b"2 3\n101\n010\n"
    w, n, f = fio.read_matrix_host(p)
    assert f == fio.Format.ascii and (w == a).all()
    # test_io.cpp:23-39 binary layout
    b = np.array([[1, 1]], np.uint64)
    p = tmp_path / "b.bmf2"
    fio.write_matrix_host(p, b, 65, fio.Format.binary)
    s = p.read_bytes()
    assert len(s) == 4 + 1 + 8 + 8 + 2 * 8
    assert s[:4] == b"BMF2" and s[4] == 1 and s[5] == 1 and s[13] == 65 and s[21] == 1 and s[29] == 1
    w, n, f = fio.read_matrix_host(p)
    assert n == 65 and (w == b).all()
    # test_io.cpp:81-89 permutation output
    p = tmp_path / "p.txt"
    fio.write_permutation(p, np.array([2, 1, 2, 3], np.uint64))
    assert p.read_bytes() == b"2 1 2 3\n" == open(os.path.join(IO, "perm4.txt"), "rb").read()
    assert list(fio.read_permutation(p)) == [2, 1, 2, 3]


def test_round_trip_lossless(fio, oracle, tmp_path):
    # test_io.cpp:41-56: ascii -> binary -> ascii, odd widths
    rng = np.random.default_rng(120)
    for t in range(40):
        m, n = int(rng.integers(0, 40)), int(rng.integers(1, 151))
        a = oracle.randomize(m, n, 0.4, int(rng.integers(1, 2 ** 62)))
        p1, p2, p3 = tmp_path / "1.txt", tmp_path / "2.bmf2", tmp_path / "3.txt"
        fio.write_matrix_host(p1, a, n, fio.Format.ascii)
        b, _, _ = fio.read_matrix_host(p1)
        fio.write_matrix_host(p2, b, n, fio.Format.binary)
        c, _, _ = fio.read_matrix_host(p2)
        fio.write_matrix_host(p3, c, n, fio.Format.ascii)
        assert p3.read_bytes() == p1.read_bytes() and (c == a).all()


MALFORMED = [b"", b"2\n", b"2 3\n101\n", b"1 3\n10\n", b"1 3\n1x1\n", b"1 2 3\n10\n", b"BMF9nonsense",
             b"BMF2\x02" + bytes(16),                     # test_io.cpp:58-79
             b"BMF2\x01" + bytes(10),                     # truncated header
             b"BMF2\x01" + (1).to_bytes(8, "little") + (3).to_bytes(8, "little") + bytes(4),  # truncated payload
             b"BMF2\x01" + (1 << 32).to_bytes(8, "little") + (1).to_bytes(8, "little"),       # dimension limit
             b"4294967296 1\n"]


def test_malformed_rejected(fio, tmp_path):
    import paper_1006_1744_b200 as f2
    for i, content in enumerate(MALFORMED):
        p = tmp_path / f"bad{i}"
        p.write_bytes(content)
        with pytest.raises(f2.FormatError):
            fio.read_matrix_host(p)
    # nonzero padding bits in a binary payload (test_io.cpp:71-78)
    good = tmp_path / "good.bmf2"
    fio.write_matrix_host(good, np.array([[1]], np.uint64), 2, fio.Format.binary)
    s = bytearray(good.read_bytes())
    s[21 + 7] = 0x80
    bad = tmp_path / "pad.bmf2"
    bad.write_bytes(bytes(s))
    with pytest.raises(f2.FormatError):
        fio.read_matrix_host(bad)
    with pytest.raises(f2.FormatError):
        fio.read_matrix_host(tmp_path / "does-not-exist")


def _ref_read(reflib, path):
    u64p = C.POINTER(C.c_uint64)
    L = reflib.lib
    L.ref_read_matrix.argtypes = [C.c_char_p, u64p, C.c_size_t, u64p, u64p, C.POINTER(C.c_int)]
    m, n, f = C.c_uint64(), C.c_uint64(), C.c_int()
    rc = L.ref_read_matrix(str(path).encode(), None, 0, C.byref(m), C.byref(n), C.byref(f))
    if rc:
        return rc, None, None, None
    w = np.zeros((m.value, words(n.value)), np.uint64)
    buf = w if w.size else np.zeros(1, np.uint64)
    rc = L.ref_read_matrix(str(path).encode(), buf.ctypes.data_as(u64p), max(w.size, 1), C.byref(m), C.byref(n),
                           C.byref(f))
    return rc, w, int(n.value), int(f.value)


def test_live_reference_mutations(fio, reflib, oracle, tmp_path):
    """Accept/reject and content agree with io::read_matrix on randomly mutated files."""
    import paper_1006_1744_b200 as f2
    rnd = random.Random(5)
    for t in range(200):
        m, n = rnd.randrange(0, 6), rnd.randrange(0, 140)
        a = oracle.randomize(m, n, 0.5, rnd.randrange(1, 2 ** 62))
        fmt = fio.Format(t % 2)
        p = tmp_path / "x"
        fio.write_matrix_host(p, a, n, fmt)
        s = bytearray(p.read_bytes())
        for _ in range(rnd.randrange(0, 3)):
            if not s:
                break
            k = rnd.randrange(len(s))
            op = rnd.randrange(4)
            if op == 0:
                s[k] ^= 1 << rnd.randrange(8)
            elif op == 1:
                del s[k:]
            elif op == 2:
                s.insert(k, rnd.choice(b"01 \r\nB2x"))
            else:
                s[k] = rnd.choice(b"01 \n")
        p.write_bytes(bytes(s))
        rc, rw, rn, rf = _ref_read(reflib, p)
        if rc == 9:  # std::bad_alloc: a mutated header asked for more rows than memory holds
            fio.probe(p)
            continue
        if rc:
            assert rc == 6, rc
            with pytest.raises(f2.FormatError):
                fio.read_matrix_host(p)
        else:
            w, n2, f = fio.read_matrix_host(p)
            assert n2 == rn and int(f) == rf and (w == rw).all()
