"""Column-sharded PLS across ranks.

Rank k of N holds panels p = k, k+N, k+2N, ... (W columns each, the last one
possibly narrower) side by side in a local matrix with all m rows.  For every
panel p, in column order:

1. the owner (rank p % N) factors the panel with the engine's leaf chain — the
   Gaussian pivot rule restricted to the panel's columns is the global rule
   because every column left of p is finished — and exports a header (pivot
   columns, re-mapped row positions, P entries) plus the panel's words for the
   rows >= r (the L block that every other rank needs);
2. the header and the words are broadcast from the owner (NCCL over NVLink on
   GPUs, gloo in the CPU tests);
3. every rank applies the panel to its own columns right of p: the same row
   gather, the panel TRSM and the Schur multiply, reading L from the broadcast
   words (row operations act on every column independently, so a column shard
   needs nothing else).

P, the pivot columns and every packed column are identical to the single-GPU
engine's; :func:`gather` reassembles the packed matrix for checking/output.

The schedule is written against two small interfaces so the same code drives
real GPUs and the CPU tests: ``ops`` (per-rank compute: :class:`GpuOps` calls the
C ABI) and ``comm`` (``broadcast(buf, root)``; :class:`TorchComm` wraps
``torch.distributed``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np


def owner_of(p: int, world: int) -> int:
    return p % world


def local_panels(rank: int, world: int, npanels: int) -> List[int]:
    return list(range(rank, npanels, world))


def panel_width(p: int, n: int, W: int) -> int:
    return min(W, n - p * W)


def local_ncols(rank: int, world: int, n: int, W: int) -> int:
    npan = (n + W - 1) // W
    return sum(panel_width(p, n, W) for p in local_panels(rank, world, npan))


def local_word0(p: int, rank: int, world: int, W: int) -> int:
    """Local word index where global panel p (owned by `rank`) starts."""
    assert p % world == rank
    return (p // world) * (W // 64)


def first_trailing_word(p: int, rank: int, world: int, W: int) -> int:
    """Local word index of the first local panel with global index > p."""
    owned_upto = (p - rank) // world + 1 if p >= rank else 0  # local panels with index <= p
    return owned_upto * (W // 64)


def split_columns(words: np.ndarray, n: int, rank: int, world: int, W: int) -> np.ndarray:
    """This rank's column shard of a host matrix (reference packing), panels side by side."""
    npan = (n + W - 1) // W
    parts = [words[:, (p * W) // 64:(p * W) // 64 + (panel_width(p, n, W) + 63) // 64]
             for p in local_panels(rank, world, npan)]
    if not parts:
        return np.zeros((words.shape[0], 0), np.uint64)
    return np.ascontiguousarray(np.concatenate(parts, axis=1))


def gather(shards: List[np.ndarray], m: int, n: int, W: int) -> np.ndarray:
    """Inverse of split_columns over all ranks."""
    world = len(shards)
    npan = (n + W - 1) // W
    out = np.zeros((m, (n + 63) // 64), np.uint64)
    for k, sh in enumerate(shards):
        col = 0
        for p in local_panels(k, world, npan):
            nw = (panel_width(p, n, W) + 63) // 64
            out[:, (p * W) // 64:(p * W) // 64 + nw] = sh[:, col:col + nw]
            col += nw
    return out


@dataclass
class ShardResult:
    rank: int
    P: np.ndarray        # uint64[m] transpositions (LAPACK form)
    pivcols: np.ndarray  # uint64[rank] pivot columns (Q prefix)


def header_fields(hdr: np.ndarray, W: int, kmax_moved: int):
    kb, r0 = int(hdr[0]), int(hdr[1])
    q = hdr[4:4 + kb]
    P = hdr[4 + W + 2 * kmax_moved:4 + W + 2 * kmax_moved + kb]
    return kb, r0, q, P


def pls_sharded(ops, comm, local, m: int, n: int, W: int, rank: int, world: int) -> ShardResult:
    """Run the column-sharded PLS on this rank's local matrix (in place)."""
    npan = (n + W - 1) // W
    hdr, words = ops.exchange_buffers(m, W)
    ops.begin(local)
    r = 0
    P = np.arange(m, dtype=np.uint64)
    piv: List[int] = []
    for p in range(npan):
        if r >= m:
            break
        w = panel_width(p, n, W)
        own = owner_of(p, world)
        if rank == own:
            ops.factor_panel(local, local_word0(p, rank, world, W), w, r, p * W, hdr, words)
        comm.broadcast(hdr, own)
        comm.broadcast(words, own)
        h = ops.read_header(hdr)
        kb, r0, q, Pp = header_fields(h, W, ops.kmax_moved)
        assert r0 == r
        tw0 = first_trailing_word(p, rank, world, W)
        ops.apply_panel(local, tw0, w, rank == own, hdr, words)
        if kb:
            P[r:r + kb] = Pp
            piv.extend(int(x) + p * W for x in q)
        r += kb
    return ShardResult(r, P, np.asarray(piv, dtype=np.uint64))


# --------------------------------------------------------------------------- GPU side
class GpuOps:
    """Per-rank compute through the C ABI (f2_dist_*)."""

    def __init__(self, f2):
        self.f2 = f2
        L = self.L = f2.load_library()
        sz, vp, u64 = C.c_size_t, C.c_void_p, C.c_uint64
        L.f2_dist_header_words.argtypes = [C.c_uint]
        L.f2_dist_header_words.restype = sz
        L.f2_dist_begin.argtypes = [vp]
        L.f2_dist_factor_panel.argtypes = [vp, sz, C.c_uint, u64, u64, vp, vp, sz, C.POINTER(u64)]
        L.f2_dist_apply_panel.argtypes = [vp, sz, C.c_uint, C.c_int, vp, vp, sz]
        L.f2_device_alloc.argtypes = [sz]
        L.f2_device_alloc.restype = vp
        L.f2_device_free.argtypes = [vp]
        L.f2_device_copy.argtypes = [vp, vp, sz, C.c_int]
        self.kmax_moved = (int(L.f2_dist_header_words(0)) - 4) // 2

    def exchange_buffers(self, m: int, W: int):
        """Header + words buffers.  Torch CUDA tensors when torch is used for the
        exchange (comm needs them), raw device buffers otherwise."""
        self.W = W
        self.words_stride = W // 64
        hw = int(self.L.f2_dist_header_words(W))
        try:
            import torch
            if torch.cuda.is_available():
                self._hdr = torch.zeros(hw, dtype=torch.int64, device="cuda")
                self._words = torch.zeros(m * self.words_stride, dtype=torch.int64, device="cuda")
                return self._hdr, self._words
        except Exception:
            pass
        raise RuntimeError("GpuOps needs torch CUDA tensors for the exchange buffers")

    @staticmethod
    def _ptr(t):
        return C.c_void_p(t.data_ptr())

    def begin(self, local):
        self.f2._check(self.L.f2_dist_begin(local.handle))

    def factor_panel(self, local, pw0, width, r, panel_col, hdr, words):
        kb = C.c_uint64()
        self.f2._check(self.L.f2_dist_factor_panel(local.handle, pw0, width, r, panel_col, self._ptr(hdr),
                                                   self._ptr(words), self.words_stride, C.byref(kb)))
        return int(kb.value)

    def apply_panel(self, local, tw0, width, owner, hdr, words):
        self.f2._check(self.L.f2_dist_apply_panel(local.handle, tw0, width, int(owner), self._ptr(hdr),
                                                  self._ptr(words), self.words_stride))

    def read_header(self, hdr):
        return hdr.cpu().numpy().view(np.uint64)


class TorchComm:
    """broadcast over torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def broadcast(self, buf, root: int):
        self.dist.broadcast(buf, src=root, group=self.group)


class LocalComm:
    """Single-process emulation: all ranks share the exchange buffers."""

    def broadcast(self, buf, root: int):
        return None


def pls_sharded_emulated(ops, locals_: list, m: int, n: int, W: int) -> ShardResult:
    """All ranks in one process on one device, panel by panel (owner factors, owner
    applies, then every other rank applies) — the schedule pls_sharded runs with one
    process per GPU, with the broadcast replaced by shared exchange buffers."""
    world = len(locals_)
    npan = (n + W - 1) // W
    hdr, words = ops.exchange_buffers(m, W)
    ops.begin(locals_[0])
    r = 0
    P = np.arange(m, dtype=np.uint64)
    piv: List[int] = []
    for p in range(npan):
        if r >= m:
            break
        w = panel_width(p, n, W)
        own = owner_of(p, world)
        ops.factor_panel(locals_[own], local_word0(p, own, world, W), w, r, p * W, hdr, words)
        kb, r0, q, Pp = header_fields(ops.read_header(hdr), W, ops.kmax_moved)
        for k in [own] + [x for x in range(world) if x != own]:
            ops.apply_panel(locals_[k], first_trailing_word(p, k, world, W), w, k == own, hdr, words)
        if kb:
            P[r:r + kb] = Pp
            piv.extend(int(x) + p * W for x in q)
        r += kb
    return ShardResult(r, P, np.asarray(piv, dtype=np.uint64))
