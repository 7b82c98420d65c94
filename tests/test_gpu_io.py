"""GPU: BMF2/ASCII load straight into HBM and store straight from it (csrc/io.cu),
against the reference-written fixtures (tests/golden/io/) and through a
read -> PLS -> RREF -> write pipeline; chunk boundaries forced small."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
IO = os.path.join(HERE, "golden", "io")


@pytest.fixture(scope="module")
def fio(f2):
    from paper_1006_1744_b200 import io
    return io


def test_golden_load_store(f2, fio, tmp_path):
    z = np.load(os.path.join(IO, "matrices.npz"))
    for i in range(int(z["count"])):
        a, n = z[f"m{i}"], int(z[f"n{i}"])
        for ext, fmt in [("txt", fio.Format.ascii), ("bmf2", fio.Format.binary)]:
            p = os.path.join(IO, f"mat{i}_{a.shape[0]}x{n}.{ext}")
            d, f = fio.read_matrix(p)
            assert f == fmt and d.nrows == a.shape[0] and d.ncols == n
            if a.size:
                assert (d.download() == a).all()
            out = tmp_path / f"o.{ext}"
            fio.write_matrix(out, d, fmt)
            assert out.read_bytes() == open(p, "rb").read()


@pytest.mark.parametrize("chunk", [0, 8, 4096, 1 << 20])
def test_streaming_chunks(f2, fio, oracle, tmp_path, monkeypatch, chunk):
    """Chunked pinned double-buffer pipeline: every chunk size gives the same bytes."""
    if chunk:
        monkeypatch.setenv("F2_IO_CHUNK_BYTES", str(chunk))
    m, n = 3001, 4161
    a = oracle.randomize(m, n, 0.5, 99)
    p = tmp_path / "a.bmf2"
    fio.write_matrix_host(p, a, n, fio.Format.binary)
    d, f = fio.read_matrix(p)
    assert f == fio.Format.binary and (d.download() == a).all()
    q = tmp_path / "b.bmf2"
    fio.write_matrix(q, d, fio.Format.binary)
    assert q.read_bytes() == p.read_bytes()


def test_load_errors(f2, fio, tmp_path):
    bad = tmp_path / "bad.bmf2"
    s = bytearray(b"BMF2\x01" + (3).to_bytes(8, "little") + (2).to_bytes(8, "little") + bytes(24))
    s[21 + 8 + 7] = 0x80  # padding bit of row 1
    bad.write_bytes(bytes(s))
    with pytest.raises(f2.FormatError):
        fio.read_matrix(bad)
    bad.write_bytes(bytes(s[:30]))
    with pytest.raises(f2.FormatError):
        fio.read_matrix(bad)


def test_pipeline_file_to_rref(f2, fio, oracle, tmp_path):
    m, n = 1500, 2300
    a = oracle.randomize(m, n, 0.3, 5)
    p = tmp_path / "in.bmf2"
    fio.write_matrix_host(p, a, n, fio.Format.binary)
    d, _ = fio.read_matrix(p)
    r = f2.rref(d)
    want, wr = oracle.gauss_rref(a, n)
    assert r == wr
    out = tmp_path / "out.txt"
    fio.write_matrix(out, d, fio.Format.ascii)
    got, n2, fmt = fio.read_matrix_host(out)
    assert fmt == fio.Format.ascii and n2 == n and (got == want).all()
