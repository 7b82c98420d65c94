"""On-disk formats — mirror of ``f2lin::io`` (proj/include/f2lin/io.hpp, src/io.cpp).

Binary "BMF2" (magic, version 0x01, u64 LE nrows/ncols, row-major u64 LE words,
padding zero) and ASCII ("<nrows> <ncols>" then rows of 0/1).  Everything is in
the native library (paper_1006_1744_b200/csrc/io.cu): ``read_matrix`` streams a
binary payload straight into HBM through pinned double buffers; the ``*_host``
variants and the permutation functions need no GPU.  Malformed input raises
:class:`FormatError` exactly where io.cpp throws ``io::FormatError``.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from typing import Tuple, Union

import numpy as np

from . import (DeviceMatrix, FormatError, _check, _ptr, host_words, load_library)

__all__ = ["Format", "FormatError", "read_matrix", "write_matrix", "read_matrix_host", "write_matrix_host",
           "probe", "read_permutation", "write_permutation"]

PathLike = Union[str, os.PathLike]


class Format(enum.IntEnum):
    """io::Format (io.hpp:22)."""
    ascii = 0
    binary = 1


def _p(path: PathLike) -> bytes:
    return os.fsencode(path)


def probe(path: PathLike) -> Tuple[int, int, Format]:
    """(nrows, ncols, format) from the header (format sniffed as io.cpp:118-126)."""
    L = load_library()
    m, n, f = C.c_uint64(), C.c_uint64(), C.c_int()
    _check(L.f2_io_probe(_p(path), C.byref(m), C.byref(n), C.byref(f)))
    return int(m.value), int(n.value), Format(f.value)


def read_matrix_host(path: PathLike) -> Tuple[np.ndarray, int, Format]:
    """io::read_matrix(path, &detected) into host words (reference packing)."""
    L = load_library()
    m, n, fmt = probe(path)
    w = np.zeros((m, host_words(n)), np.uint64)
    _check(L.f2_io_read_host(_p(path), _ptr(w) if w.size else None, w.shape[1], m, n))
    return w, n, fmt


def write_matrix_host(path: PathLike, words: np.ndarray, ncols: int, fmt: Format = Format.binary) -> None:
    """io::write_matrix(path, a, fmt) from host words."""
    L = load_library()
    w = np.ascontiguousarray(words, dtype=np.uint64)
    stride = w.shape[1] if w.ndim == 2 and w.shape[0] else host_words(ncols)
    _check(L.f2_io_write_host(_p(path), _ptr(w) if w.size else None, stride, w.shape[0], ncols, int(fmt)))


def read_matrix(path: PathLike) -> Tuple[DeviceMatrix, Format]:
    """io::read_matrix(path, &detected) straight into an HBM-resident matrix."""
    L = load_library()
    h, f = C.c_void_p(), C.c_int()
    _check(L.f2_matrix_load(_p(path), C.byref(h), C.byref(f)))
    out = DeviceMatrix.__new__(DeviceMatrix)
    out._h = h
    out.nrows, out.ncols = int(L.f2_matrix_nrows(h)), int(L.f2_matrix_ncols(h))
    return out, Format(f.value)


def write_matrix(path: PathLike, a: DeviceMatrix, fmt: Format = Format.binary) -> None:
    """io::write_matrix(path, a, fmt) straight from HBM."""
    _check(load_library().f2_matrix_store(a.handle, _p(path), int(fmt)))


def write_permutation(path: PathLike, p: np.ndarray) -> None:
    """io::write_permutation: one line of space-separated entries."""
    p = np.ascontiguousarray(p, dtype=np.uint64)
    _check(load_library().f2_write_permutation(_p(path), _ptr(p) if p.size else None, p.size))


def read_permutation(path: PathLike) -> np.ndarray:
    """io::read_permutation: the entries of the first line."""
    L = load_library()
    n = C.c_size_t()
    _check(L.f2_read_permutation(_p(path), None, 0, C.byref(n)))
    out = np.zeros(n.value, np.uint64)
    if n.value:
        _check(L.f2_read_permutation(_p(path), _ptr(out), out.size, C.byref(n)))
    return out
