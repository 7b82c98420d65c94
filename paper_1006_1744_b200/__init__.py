"""B200-native GF(2) PLS decomposition — host-side mirror of the reference API.

The reference (`f2lin`, /root/reference/proj/include/f2lin) is a C++ library;
this package is a thin ctypes layer over the C ABI in ``include/f2lin_gpu.h``
(``libf2gpu.so``: C++ host orchestration + sm_100a CUDA kernels).  Names,
argument meaning and error behaviour follow the reference:

==========================  ==============================================  ==========================
this module                 reference                                        raises (reference)
==========================  ==============================================  ==========================
DeviceMatrix                BitMatrix (bitmat.hpp:90-234), in HBM            --
DeviceMatrix.window         MatrixWindow (bitmat.hpp:239-330)                IndexError (out_of_range)
DeviceMatrix.randomize      BitMatrix::randomize (bitmat.cpp:136-154)        ValueError (invalid_argument)
mmpf_pls                    mmpf_pls (mmpf.hpp:35-37)                        ValueError
pls_recursive               pls_recursive (pls.hpp:42-47)                    ValueError
addmul / mul_m4rm           addmul / mul_m4rm (mul.hpp:17-20)                ValueError
trsm_lower_left_unit        trsm_lower_left_unit (mul.hpp:24)                ValueError
compress_columns            compress_columns (perm.hpp:61)                   ValueError
apply_rows                  Permutation::apply_rows[_inverse] (perm.hpp:42)  ValueError
EliminationConfig           EliminationConfig (pls.hpp:26-35)                --
PlsResult                   PlsResult (gauss.hpp:22-26)                      --
==========================  ==============================================  ==========================

There is no CPU fallback: every compute call goes to the CUDA library and fails
loudly (``NoDeviceError``) when no B200 is visible or the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "load_library", "DeviceMatrix", "Window", "EliminationConfig", "PlsResult", "mmpf_pls", "pls_recursive",
    "mmpf_pls_host", "pls_recursive_host", "addmul", "mul_m4rm", "trsm_lower_left_unit", "compress_columns",
    "apply_rows", "default_cutoff_bytes", "auto_table_bits", "NoDeviceError", "F2Error", "host_words",
    "pinned_empty", "stats_enable", "stats_get", "stats_reset", "last_launch_count", "set_panel_bits",
    "timer_start", "timer_stop", "set_device", "rref_from_pls", "rref", "FormatError",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# F2_LIB: an alternative build of the same library (A/B timing tools only)
LIB_PATH = os.environ.get("F2_LIB") or os.path.join(_HERE, "libf2gpu.so")

F2_OK, F2_INVALID_ARGUMENT, F2_OUT_OF_RANGE, F2_CUDA_ERROR, F2_NO_DEVICE, F2_OUT_OF_MEMORY, F2_FORMAT_ERROR = range(7)
ALG_GAUSS, ALG_M4RI, ALG_MMPF, ALG_PLS, ALG_HYBRID = range(5)


class F2Error(RuntimeError):
    pass


class NoDeviceError(F2Error):
    pass


class FormatError(F2Error):
    """io::FormatError (io.hpp:24-26)."""


class _Window(C.Structure):
    _fields_ = [("r0", C.c_size_t), ("c0", C.c_size_t), ("r1", C.c_size_t), ("c1", C.c_size_t)]


class _Cfg(C.Structure):
    _fields_ = [("k", C.c_uint), ("cutoff_bytes", C.c_uint64), ("hybrid_threshold", C.c_double),
                ("algorithm", C.c_int)]


_u64p = C.POINTER(C.c_uint64)
_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libf2gpu.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NoDeviceError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    sz, vp, i = C.c_size_t, C.c_void_p, C.c_int
    sig = {
        "f2_last_error": ([], C.c_char_p),
        "f2_device_count": ([], i),
        "f2_set_device": ([i], i),
        "f2_matrix_create": ([sz, sz, C.POINTER(vp)], i),
        "f2_matrix_destroy": ([vp], None),
        "f2_matrix_nrows": ([vp], sz),
        "f2_matrix_ncols": ([vp], sz),
        "f2_matrix_stride": ([vp], sz),
        "f2_matrix_device_ptr": ([vp], _u64p),
        "f2_matrix_view": ([_u64p, sz, sz, sz, C.POINTER(vp)], i),
        "f2_matrix_upload": ([vp, _u64p, sz], i),
        "f2_matrix_download": ([vp, _u64p, sz], i),
        "f2_matrix_copy": ([vp, vp], i),
        "f2_matrix_clear": ([vp], i),
        "f2_matrix_randomize": ([vp, C.c_double, C.c_uint64], i),
        "f2_matrix_digest": ([vp, _u64p], i),
        "f2_matrix_fixed_weight": ([vp, sz, C.c_uint64], i),
        "f2_host_alloc": ([sz], vp),
        "f2_host_free": ([vp], None),
        "f2_mmpf_pls": ([vp, _Window, _u64p, sz, _u64p, sz, C.c_uint, _u64p], i),
        "f2_pls_recursive": ([vp, _Window, _u64p, sz, _u64p, sz, C.POINTER(_Cfg), _u64p], i),
        "f2_mmpf_pls_host": ([_u64p, sz, sz, sz, _u64p, _u64p, C.c_uint, _u64p], i),
        "f2_pls_recursive_host": ([_u64p, sz, sz, sz, _u64p, _u64p, C.POINTER(_Cfg), _u64p], i),
        "f2_rref_from_pls": ([vp, _Window, C.c_uint64, _u64p, sz], i),
        "f2_rref": ([vp, _Window, C.POINTER(_Cfg), _u64p], i),
        "f2_default_cutoff_bytes": ([], C.c_uint64),
        "f2_io_probe": ([C.c_char_p, _u64p, _u64p, C.POINTER(i)], i),
        "f2_io_read_host": ([C.c_char_p, _u64p, sz, C.c_uint64, C.c_uint64], i),
        "f2_io_write_host": ([C.c_char_p, _u64p, sz, C.c_uint64, C.c_uint64, i], i),
        "f2_matrix_load": ([C.c_char_p, C.POINTER(vp), C.POINTER(i)], i),
        "f2_matrix_store": ([vp, C.c_char_p, i], i),
        "f2_write_permutation": ([C.c_char_p, _u64p, sz], i),
        "f2_read_permutation": ([C.c_char_p, _u64p, sz, C.POINTER(sz)], i),
        "f2_auto_table_bits": ([sz], C.c_uint),
        "f2_addmul": ([vp, _Window, vp, _Window, vp, _Window, C.c_uint], i),
        "f2_mul_m4rm": ([vp, vp, C.c_uint, C.POINTER(vp)], i),
        "f2_trsm_lower_left_unit": ([vp, _Window, vp, _Window], i),
        "f2_trsm_upper_left_unit": ([vp, _Window, vp, _Window], i),
        "f2_compress_columns": ([vp, C.c_uint64, _u64p, sz], i),
        "f2_apply_rows": ([vp, _Window, _u64p, sz, i], i),
        "f2_stats_enable": ([i], i),
        "f2_stats_get": ([i, _u64p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)], i),
        "f2_stats_reset": ([], i),
        "f2_m4ri_rref": ([vp, C.c_uint, i, C.POINTER(C.c_uint64)], i),
        "f2_hybrid_rref": ([vp, C.POINTER(_Cfg), C.POINTER(C.c_uint64)], i),
        "f2_rank": ([vp, C.POINTER(_Cfg), C.POINTER(C.c_uint64)], i),
        "f2_last_launch_count": ([], C.c_uint64),
        "f2_last_graph_kernels": ([], C.c_uint64),
        "f2_set_panel_bits": ([C.c_uint], i),
        "f2_timer_start": ([], i),
        "f2_timer_stop": ([C.POINTER(C.c_double)], i),
        "f2_debug_clocks": ([C.POINTER(C.c_longlong), i], i),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("F2_LIB") and not hasattr(L, name):
            continue  # A/B timing against an older build: skip entry points it lacks
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == F2_OK:
        return
    msg = (_lib.f2_last_error() or b"").decode()
    if rc == F2_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == F2_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == F2_NO_DEVICE:
        raise NoDeviceError(msg)
    if rc == F2_OUT_OF_MEMORY:
        raise MemoryError(msg)
    if rc == F2_FORMAT_ERROR:
        raise FormatError(msg)
    raise F2Error(f"CUDA error: {msg}")


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def host_words(ncols: int) -> int:
    """Words per row in the reference packing (bitmat.hpp:94-98)."""
    return (ncols + 63) // 64


class _PinnedOwner:
    def __init__(self, lib, ptr):
        self.lib, self.ptr = lib, ptr

    def __del__(self):
        try:
            self.lib.f2_host_free(self.ptr)
        except Exception:
            pass


def pinned_empty(shape, dtype=np.uint64) -> np.ndarray:
    """numpy array over page-locked host memory (for timed host<->device copies);
    the memory is released when the array (and its views) are gone."""
    L = load_library()
    count = int(np.prod(shape))
    nbytes = max(count * np.dtype(dtype).itemsize, 8)
    p = L.f2_host_alloc(nbytes)
    if not p:
        raise MemoryError("cudaMallocHost failed")
    buf = (C.c_char * nbytes).from_address(p)
    buf._owner = _PinnedOwner(L, p)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)




@dataclass
class Window:
    """MatrixWindow bounds (half-open), bitmat.hpp:239-250."""
    r0: int
    c0: int
    r1: int
    c1: int

    def c(self) -> _Window:
        return _Window(self.r0, self.c0, self.r1, self.c1)


@dataclass
class EliminationConfig:
    """pls.hpp:26-35."""
    k: int = 0
    cutoff_bytes: int = 0
    hybrid_threshold: float = 0.15
    algorithm: int = ALG_PLS

    def c(self) -> _Cfg:
        return _Cfg(self.k, self.cutoff_bytes, self.hybrid_threshold, self.algorithm)

    def effective_cutoff(self) -> int:
        return self.cutoff_bytes or default_cutoff_bytes()


@dataclass
class PlsResult:
    """gauss.hpp:22-26: rank plus the transposition vectors P (m) and Q (n)."""
    rank: int = 0
    P: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    Q: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


class DeviceMatrix:
    """A BitMatrix resident in B200 HBM (rows padded to 128 B)."""

    def __init__(self, nrows: int, ncols: int):
        L = load_library()
        h = C.c_void_p()
        _check(L.f2_matrix_create(nrows, ncols, C.byref(h)))
        self._h = h
        self.nrows, self.ncols = nrows, ncols

    @classmethod
    def from_host(cls, words: np.ndarray, ncols: int) -> "DeviceMatrix":
        a = cls(words.shape[0], ncols)
        a.upload(words)
        return a

    @staticmethod
    def stride_for(ncols: int) -> int:
        """Row stride in words: ceil(ncols / 64) padded to 16 words (128 B)."""
        return (host_words(ncols) + 15) // 16 * 16

    @classmethod
    def from_torch(cls, t, ncols: int) -> "DeviceMatrix":
        """A matrix over the memory of a CUDA tensor of shape (m, stride_for(ncols)), int64
        (f2_matrix_view; the tensor is kept alive by the matrix).  Padding words must be 0."""
        assert t.is_cuda and t.dim() == 2 and t.is_contiguous() and t.element_size() == 8
        assert t.shape[1] % 16 == 0 and t.shape[1] >= host_words(ncols)
        L = load_library()
        h = C.c_void_p()
        _check(L.f2_matrix_view(C.cast(C.c_void_p(t.data_ptr()), _u64p), t.shape[0], ncols, t.shape[1], C.byref(h)))
        a = cls.__new__(cls)
        a._h = h
        a.nrows, a.ncols = int(t.shape[0]), ncols
        a.tensor = t
        return a

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.f2_matrix_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def stride(self) -> int:
        return int(_lib.f2_matrix_stride(self._h))

    def upload(self, words: np.ndarray) -> None:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        assert w.shape[0] == self.nrows and (self.nrows == 0 or w.shape[1] >= host_words(self.ncols))
        _check(_lib.f2_matrix_upload(self._h, _ptr(w), w.shape[1] if w.ndim == 2 else host_words(self.ncols)))

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.zeros((self.nrows, host_words(self.ncols)), dtype=np.uint64)
        _check(_lib.f2_matrix_download(self._h, _ptr(out), out.shape[1]))
        return out

    def randomize(self, density: float, seed: int) -> None:
        _check(_lib.f2_matrix_randomize(self._h, float(density), int(seed) & (2 ** 64 - 1)))

    def fixed_weight(self, weight: int, seed: int) -> None:
        """Every row gets exactly ``weight`` ones at distinct uniform columns (config 5)."""
        _check(_lib.f2_matrix_fixed_weight(self._h, int(weight), int(seed) & (2 ** 64 - 1)))

    def clear(self) -> None:
        _check(_lib.f2_matrix_clear(self._h))

    def copy_from(self, other: "DeviceMatrix") -> None:
        _check(_lib.f2_matrix_copy(self._h, other._h))

    def clone(self) -> "DeviceMatrix":
        b = DeviceMatrix(self.nrows, self.ncols)
        b.copy_from(self)
        return b

    def digest(self) -> int:
        out = C.c_uint64()
        _check(_lib.f2_matrix_digest(self._h, C.byref(out)))
        return int(out.value)

    def view(self) -> Window:
        return Window(0, 0, self.nrows, self.ncols)

    def window(self, r0: int, c0: int, r1: int, c1: int) -> Window:
        if r0 > r1 or c0 > c1 or r1 > self.nrows or c1 > self.ncols:
            raise IndexError("MatrixWindow: invalid bounds")
        return Window(r0, c0, r1, c1)


def _win(a: DeviceMatrix, w: Optional[Window]) -> Window:
    return a.view() if w is None else w


def mmpf_pls(a: DeviceMatrix, k: int = 0, window: Optional[Window] = None) -> PlsResult:
    """In-place MMPF PLS of ``a`` (or a window of it); mmpf.hpp:35-37."""
    w = _win(a, window)
    m, n = w.r1 - w.r0, w.c1 - w.c0
    p = np.zeros(max(m, 0), np.uint64)
    q = np.zeros(max(n, 0), np.uint64)
    r = C.c_uint64()
    _check(_lib.f2_mmpf_pls(a.handle, w.c(), _ptr(p), p.size, _ptr(q), q.size, k, C.byref(r)))
    return PlsResult(int(r.value), p, q)


def pls_recursive(a: DeviceMatrix, cfg: Optional[EliminationConfig] = None,
                  window: Optional[Window] = None) -> PlsResult:
    """In-place recursive PLS; pls.hpp:42-47.  Q (tail included) matches the
    reference's recursion for the configured cutoff."""
    cfg = cfg or EliminationConfig()
    w = _win(a, window)
    m, n = w.r1 - w.r0, w.c1 - w.c0
    p = np.zeros(max(m, 0), np.uint64)
    q = np.zeros(max(n, 0), np.uint64)
    r = C.c_uint64()
    cc = cfg.c()
    _check(_lib.f2_pls_recursive(a.handle, w.c(), _ptr(p), p.size, _ptr(q), q.size, C.byref(cc), C.byref(r)))
    return PlsResult(int(r.value), p, q)


def rref_from_pls(a: DeviceMatrix, rank: int, q: np.ndarray, window: Optional[Window] = None,
                  p: Optional[np.ndarray] = None) -> None:
    """Reduced row echelon form from a packed PLS result, in place; pls.hpp:54-59,
    pls.cpp:128-161.  ``q`` is the pivot-column prefix (Q[:rank] or all of Q);
    ``p``, when given, is only length-checked like the BitMatrix overload (pls.cpp:157-161)."""
    w = _win(a, window)
    if p is not None and len(p) != w.r1 - w.r0:
        raise ValueError("rref_from_pls: P has the wrong length")
    q = np.ascontiguousarray(q, dtype=np.uint64)
    if p is not None:
        q = q[:min(q.size, rank)].copy()
    _check(_lib.f2_rref_from_pls(a.handle, w.c(), rank, _ptr(q), q.size))


def rref(a: DeviceMatrix, cfg: Optional[EliminationConfig] = None, window: Optional[Window] = None) -> int:
    """Echelonize in place (pls_recursive + rref_from_pls, the reference's Algorithm::pls
    RREF, acceptance.cpp:37-41); returns the rank.  Equals gauss_rref bit for bit."""
    cc = (cfg or EliminationConfig()).c()
    r = C.c_uint64()
    _check(_lib.f2_rref(a.handle, _win(a, window).c(), C.byref(cc), C.byref(r)))
    return int(r.value)


def m4ri_rref(a: DeviceMatrix, k: int = 0, full: bool = True) -> int:
    """In-place M4RI elimination (m4ri.hpp:41): the RREF, or with full=False M4RI's echelon
    form; returns the rank."""
    r = C.c_uint64()
    _check(_lib.f2_m4ri_rref(a.handle, k, int(full), C.byref(r)))
    return int(r.value)


def hybrid_rref(a: DeviceMatrix, cfg: Optional[EliminationConfig] = None) -> int:
    """hybrid_rref (pls.hpp:61): in-place RREF; returns the rank."""
    r = C.c_uint64()
    cc = (cfg or EliminationConfig(algorithm=ALG_HYBRID)).c()
    _check(_lib.f2_hybrid_rref(a.handle, C.byref(cc), C.byref(r)))
    return int(r.value)


def rank(a: DeviceMatrix, cfg: Optional[EliminationConfig] = None) -> int:
    """rank(const BitMatrix&, cfg) (pls.hpp:64); A is not modified."""
    r = C.c_uint64()
    cc = (cfg or EliminationConfig()).c()
    _check(_lib.f2_rank(a.handle, C.byref(cc), C.byref(r)))
    return int(r.value)


def _pls_host(fn, words, ncols, extra):
    load_library()
    w = words
    assert w.dtype == np.uint64 and w.flags["C_CONTIGUOUS"]
    m = w.shape[0]
    p = np.zeros(m, np.uint64)
    q = np.zeros(ncols, np.uint64)
    r = C.c_uint64()
    _check(fn(_ptr(w), m, ncols, w.shape[1] if m else host_words(ncols), _ptr(p), _ptr(q), extra, C.byref(r)))
    return PlsResult(int(r.value), p, q)


def mmpf_pls_host(words: np.ndarray, ncols: int, k: int = 0) -> PlsResult:
    """Host-buffer MMPF: upload, decompose, download (``words`` updated in place)."""
    return _pls_host(load_library().f2_mmpf_pls_host, words, ncols, k)


def pls_recursive_host(words: np.ndarray, ncols: int, cfg: Optional[EliminationConfig] = None) -> PlsResult:
    cc = (cfg or EliminationConfig()).c()
    return _pls_host(load_library().f2_pls_recursive_host, words, ncols, C.byref(cc))


def addmul(c: DeviceMatrix, a: DeviceMatrix, b: DeviceMatrix, k: int = 0, wc: Optional[Window] = None,
           wa: Optional[Window] = None, wb: Optional[Window] = None) -> None:
    """C ^= A*B over windows (mul.hpp:20); C must not alias A or B."""
    _check(_lib.f2_addmul(c.handle, _win(c, wc).c(), a.handle, _win(a, wa).c(), b.handle, _win(b, wb).c(), k))


def mul_m4rm(a: DeviceMatrix, b: DeviceMatrix, k: int = 0) -> DeviceMatrix:
    """mul.hpp:17."""
    h = C.c_void_p()
    _check(_lib.f2_mul_m4rm(a.handle, b.handle, k, C.byref(h)))
    out = DeviceMatrix.__new__(DeviceMatrix)
    out._h = h
    out.nrows, out.ncols = a.nrows, b.ncols
    return out


def trsm_lower_left_unit(l: DeviceMatrix, b: DeviceMatrix, wl: Optional[Window] = None,
                         wb: Optional[Window] = None) -> None:
    """B <- L^{-1} B, L unit lower (upper part ignored); mul.hpp:24."""
    _check(_lib.f2_trsm_lower_left_unit(l.handle, _win(l, wl).c(), b.handle, _win(b, wb).c()))


def trsm_upper_left_unit(u: DeviceMatrix, b: DeviceMatrix, wu: Optional[Window] = None,
                         wb: Optional[Window] = None) -> None:
    """B <- U^{-1} B, U unit upper (lower part ignored); mul.hpp:28."""
    _check(_lib.f2_trsm_upper_left_unit(u.handle, _win(u, wu).c(), b.handle, _win(b, wb).c()))


def compress_columns(a: DeviceMatrix, rank: int, q: np.ndarray) -> None:
    """perm.hpp:61."""
    q = np.ascontiguousarray(q, dtype=np.uint64)
    _check(_lib.f2_compress_columns(a.handle, rank, _ptr(q), q.size))


def apply_rows(a: DeviceMatrix, p: np.ndarray, inverse: bool = False, window: Optional[Window] = None) -> None:
    """Permutation::apply_rows / apply_rows_inverse (perm.hpp:42-45)."""
    p = np.ascontiguousarray(p, dtype=np.uint64)
    _check(_lib.f2_apply_rows(a.handle, _win(a, window).c(), _ptr(p), p.size, int(bool(inverse))))


def default_cutoff_bytes() -> int:
    return int(load_library().f2_default_cutoff_bytes())


def auto_table_bits(dim: int) -> int:
    return int(load_library().f2_auto_table_bits(dim))


def stats_enable(on: bool = True) -> None:
    _check(load_library().f2_stats_enable(int(on)))


def stats_reset() -> None:
    _check(load_library().f2_stats_reset())


def stats_get(kind: int) -> dict:
    n = C.c_uint64()
    ms, by, bo = C.c_double(), C.c_double(), C.c_double()
    _check(load_library().f2_stats_get(kind, C.byref(n), C.byref(ms), C.byref(by), C.byref(bo)))
    return dict(launches=int(n.value), ms=ms.value, bytes=by.value, bitops=bo.value)


def last_launch_count() -> int:
    return int(load_library().f2_last_launch_count())


def last_graph_kernels() -> int:
    """Kernel nodes of the CUDA graph the last graph-replayed PLS launched (0 if none)."""
    return int(load_library().f2_last_graph_kernels())


def timer_start() -> None:
    """Record a CUDA event on the library's stream."""
    _check(load_library().f2_timer_start())


def timer_stop() -> float:
    """Record a second event, wait for it, return device milliseconds since timer_start()."""
    ms = C.c_double()
    _check(load_library().f2_timer_stop(C.byref(ms)))
    return ms.value


def set_device(device: int) -> None:
    _check(load_library().f2_set_device(device))


def set_panel_bits(bits: int) -> None:
    _check(load_library().f2_set_panel_bits(bits))
