"""Column-sharded PLS across ranks, one process per GPU.

The reference has no distributed path; this is ``pls_recursive`` (pls.hpp:42-47,
pls.cpp:63-103) split by columns.  Rank k of N holds panels p = k, k+N, k+2N, ...
(W columns each, the last one possibly narrower) side by side in a local matrix
with all m rows.  For every panel p, in column order:

1. the owner (rank p % N) factors the panel (``f2_dist_factor``: the engine's panel
   kernel; the Gaussian pivot rule restricted to the panel's columns is the global
   rule because every column left of p is finished) and exports its header (pivot
   columns, P entries, re-mapped rows) and its words for the rows >= r into an
   exchange buffer;
2. the buffer's tail is broadcast from the owner (NCCL over NVLink on GPUs; gloo,
   staged through host memory, in the tests);
3. every rank applies the panel to its own columns right of p (``f2_dist_step``):
   the same row gather, panel TRSM and Schur multiply as the single-GPU engine,
   reading L from the broadcast words.

Look-ahead: the owner of panel p+1 updates panel p+1's columns first and factors
p+1 on a side stream while it updates the rest of its columns, so the broadcast of
p+1 leaves while every rank is still busy with p.  Every GPU call only enqueues on
this rank's streams: the host never waits on the GPU per panel.  It does read, three
panels late, the (kb, panel_r) of a header (``f2_dist_header_rk``) -- all ranks see
the same headers, so they agree on where each broadcast may start (rows below
panel_r are never read) and on when every row is a pivot and the loop can stop.

P, the pivot columns and every packed column are identical to the single-GPU
engine's; :func:`compress_sharded` applies ``compress_columns`` (perm.cpp:18-21)
across shards and :func:`recursive_q` replays ``pls_recursive``'s full Q
(pls.cpp:96-98) from the pivot columns.

The schedule is written against two small interfaces so the same code drives real
GPUs and the CPU tests: ``ops`` (per-rank compute; :class:`GpuOps` calls the C ABI)
and ``comm`` (``broadcast(buf, root)``; :class:`TorchComm` wraps ``torch.distributed``).
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass
from typing import List

import numpy as np

LAG = 3  # panels between a header and the host reading its (kb, panel_r)
KMAX_MOVED = 8192  # kMaxMoved (csrc/f2gpu.cuh): re-mapped positions one header carries


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


def header_offset(m: int, W: int) -> int:
    """Word offset of the header in an exchange buffer (after m rows of W/64 words)."""
    return m * (W // 64)


def header_words(W: int) -> int:
    return 4 + 2 * W + 2 * KMAX_MOVED


@dataclass
class ShardResult:
    rank: int
    P: np.ndarray        # uint64[m] transpositions (LAPACK form)
    pivcols: np.ndarray  # uint64[rank] pivot columns (Q prefix)


def pls_sharded(ops, comm, local, m: int, n: int, W: int, rank: int, world: int) -> ShardResult:
    """Run the column-sharded PLS on this rank's local matrix (in place).  Every rank
    calls this with the same (m, n, W, world); collectives are issued in panel order."""
    npan = (n + W - 1) // W
    ops.begin(local, m, n, W, npan)
    r_known = {}

    def r_after(p):  # first row past panel p's pivots (identical on every rank)
        if p not in r_known:
            kb, r0 = ops.header_rk(p)
            r_known[p] = r0 + kb
        return r_known[p]

    def live(p):  # panel p is processed: decided from a header LAG panels back
        return p < npan and (p < LAG or r_after(p - LAG) < m)

    def r_lo(p):  # the broadcast of panel p starts at this row (<= its panel_r)
        return 0 if p < LAG else r_after(p - LAG)

    def geometry(p):
        own = owner_of(p, world)
        return own, panel_width(p, n, W), p * W

    own0, w0, c0 = geometry(0)
    if rank == own0 and npan:
        with ops.on_main():
            ops.factor(local, 0, local_word0(0, rank, world, W), w0, c0)
            if world > 1:
                comm.broadcast(ops.slice(0, 0), own0)
            ops.note(0)
    for p in range(npan):
        if not live(p):
            break
        own, w, _ = geometry(p)
        if rank != own:
            with ops.on_comm(p):
                comm.broadcast(ops.slice(p, r_lo(p)), own)
                ops.note(p)
            ops.main_wait_comm()
        la = live(p + 1) and owner_of(p + 1, world) == rank
        nxt = geometry(p + 1) if la else (None, 0, 0)
        ops.step(local, p, rank == own, local_word0(p, rank, world, W) if rank == own else 0, w,
                 first_trailing_word(p, rank, world, W), la, nxt[1], nxt[2])
        if la:
            with ops.on_side():  # ordered after the look-ahead factorisation of p + 1
                if world > 1:
                    comm.broadcast(ops.slice(p + 1, r_lo(p + 1)), rank)
                ops.note(p + 1)
        ops.mark_free(p)
    rk, P, piv = ops.finish(local)
    return ShardResult(rk, P, piv)


def pls_sharded_emulated(ops, locals_: list, m: int, n: int, W: int) -> ShardResult:
    """All ranks in one process on one device, panel by panel on one stream: the owner
    factors, then every rank (owner first) applies -- the exchange buffer is shared
    instead of broadcast, the per-rank state is re-imported from it.  No look-ahead."""
    world = len(locals_)
    npan = (n + W - 1) // W
    widest = max(range(world), key=lambda k: local_ncols(k, world, n, W))
    ops.begin(locals_[widest], m, n, W, npan)
    r = 0
    for p in range(npan):
        if r >= m:
            break
        own = owner_of(p, world)
        w = panel_width(p, n, W)
        with ops.on_main():
            ops.factor(locals_[own], p, local_word0(p, own, world, W), w, p * W)
            ops.note(p)
        for k in [own] + [x for x in range(world) if x != own]:
            ops.step(locals_[k], p, k == own, local_word0(p, own, world, W) if k == own else 0, w,
                     first_trailing_word(p, k, world, W), False, 0, 0)
        kb, r0 = ops.header_rk(p)
        r = r0 + kb
    rk, P, piv = ops.finish(locals_[widest])
    return ShardResult(rk, P, piv)


def compress_sharded(ops, comm, local, m: int, n: int, W: int, rank: int, world: int, res: ShardResult) -> None:
    """compress_columns (perm.cpp:18-21) of the sharded packed result: it swaps columns
    j <-> Q[j] over rows >= j, and the two columns may live on different ranks.  Nothing
    moves for an identity Q prefix (dense full-rank inputs).  Otherwise every rank
    gathers the shards (one all-gather), compresses the whole matrix on its device and
    keeps its own columns."""
    if all(int(x) == t for t, x in enumerate(res.pivcols)):
        return
    ops.compress_sharded(comm, local, m, n, W, rank, world, res)


def recursive_q(f2, m: int, n: int, cutoff: int, res: ShardResult) -> np.ndarray:
    """pls_recursive's full Q (tail included, pls.cpp:96-98) from the pivot columns."""
    L = f2.load_library()
    L.f2_recursive_q.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]
    q = np.zeros(n, np.uint64)
    piv = np.ascontiguousarray(res.pivcols, dtype=np.uint64)
    u64p = C.POINTER(C.c_uint64)
    f2._check(L.f2_recursive_q(m, n, cutoff, res.rank, piv.ctypes.data_as(u64p), q.ctypes.data_as(u64p)))
    return q


# --------------------------------------------------------------------------- GPU side
class GpuOps:
    """Per-rank compute through the C ABI (f2_dist_*) on this rank's torch streams:
    ``main`` (the panel steps), ``side`` (look-ahead factorisations and their
    broadcasts, high priority) and ``comm`` (receives)."""

    def __init__(self, f2, side_ctas: int = 0):
        import torch
        self.f2, self.torch = f2, torch
        self.side_ctas = side_ctas
        L = self.L = f2.load_library()
        sz, vp, u64, i = C.c_size_t, C.c_void_p, C.c_uint64, C.c_int
        L.f2_dist_buffer_words.argtypes = [sz, C.c_uint]
        L.f2_dist_buffer_words.restype = sz
        L.f2_dist_begin.argtypes = [vp, C.c_uint, sz, vp]
        L.f2_dist_factor.argtypes = [vp, sz, C.c_uint, u64, vp, i, vp]
        L.f2_dist_step.argtypes = [vp, C.c_int64, i, sz, C.c_uint, vp, sz, i, C.c_uint, u64, vp, i, vp, vp]
        L.f2_dist_note.argtypes = [vp, C.c_int64, vp]
        L.f2_dist_header_rk.argtypes = [C.c_int64, C.POINTER(u64), C.POINTER(u64)]
        L.f2_dist_finish.argtypes = [vp, vp, C.POINTER(u64), C.POINTER(u64), sz, C.POINTER(u64), sz]
        L.f2_pls_compress.argtypes = [vp, u64, C.POINTER(u64)]
        self._cur = None

    # -- streams
    @staticmethod
    def _h(stream):
        return C.c_void_p(stream.cuda_stream)

    def _bufp(self, p):
        return C.c_void_p(self.bufs[p & 1].data_ptr())

    def begin(self, local, m, n, W, npan):
        torch = self.torch
        self.m, self.n, self.W, self.npan = m, n, W, npan
        bw = int(self.L.f2_dist_buffer_words(m, W))
        self.bufs = [torch.zeros(bw, dtype=torch.int64, device="cuda") for _ in range(2)]
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        self.main = torch.cuda.Stream()
        self.side = torch.cuda.Stream(priority=-1)
        self.comm = torch.cuda.Stream()
        cur = torch.cuda.current_stream()
        for s in (self.main, self.side, self.comm):
            s.wait_stream(cur)  # the zeroed buffers
        self.free = [None, None]
        self.f2._check(self.L.f2_dist_begin(local.handle, W, npan, self._h(self.main)))

    @contextlib.contextmanager
    def _on(self, stream):
        prev = self._cur
        self._cur = stream
        with self.torch.cuda.stream(stream):
            yield
        self._cur = prev

    def on_main(self):
        return self._on(self.main)

    def on_side(self):
        return self._on(self.side)

    def on_comm(self, p):
        ev = self.free[p & 1]
        if ev is not None:  # the buffer's previous panel (p - 2) is no longer read
            self.comm.wait_event(ev)
        return self._on(self.comm)

    def main_wait_comm(self):
        self.main.wait_stream(self.comm)

    def mark_free(self, p):
        ev = self.torch.cuda.Event()
        ev.record(self.main)
        self.free[p & 1] = ev

    def slice(self, p, r_lo):
        return self.bufs[p & 1][r_lo * (self.W // 64):]

    # -- compute
    def factor(self, local, p, pw0, width, col):
        self.f2._check(self.L.f2_dist_factor(local.handle, pw0, width, col, self._bufp(p), 0, self._h(self._cur)))

    def step(self, local, p, owner, pw0, width, tw0, lookahead, next_width, next_col):
        self.f2._check(self.L.f2_dist_step(local.handle, p, int(owner), pw0, width, self._bufp(p), tw0, int(lookahead),
                                           next_width, next_col, self._bufp(p + 1), self.side_ctas,
                                           self._h(self.main), self._h(self.side)))

    def note(self, p):
        self.f2._check(self.L.f2_dist_note(self._bufp(p), p, self._h(self._cur)))

    def header_rk(self, p):
        kb, r0 = C.c_uint64(), C.c_uint64()
        self.f2._check(self.L.f2_dist_header_rk(p, C.byref(kb), C.byref(r0)))
        return int(kb.value), int(r0.value)

    def finish(self, local):
        self.main.wait_stream(self.side)
        self.main.wait_stream(self.comm)
        P = np.zeros(self.m, np.uint64)
        piv = np.zeros(max(self.m, 1), np.uint64)
        rk = C.c_uint64()
        u64p = C.POINTER(C.c_uint64)
        self.f2._check(self.L.f2_dist_finish(local.handle, self._h(self.main), C.byref(rk), P.ctypes.data_as(u64p),
                                             P.size, piv.ctypes.data_as(u64p), piv.size))
        self.torch.cuda.current_stream().wait_stream(self.main)
        return int(rk.value), P, piv[:int(rk.value)].copy()

    def compress_sharded(self, comm, local, m, n, W, rank, world, res):
        """All-gather of the shards (torch tensors behind the local matrices), compress on
        the whole matrix (k_compress), copy this rank's columns back."""
        torch = self.torch
        npan = (n + W - 1) // W
        fstride = local.__class__.stride_for(n)
        lmax = max(local.__class__.stride_for(local_ncols(k, world, n, W)) for k in range(world))
        mine = torch.zeros((m, lmax), dtype=torch.int64, device="cuda")
        lt = local.tensor
        mine[:, :lt.shape[1]] = lt
        parts = [torch.empty_like(mine) for _ in range(world)]
        comm.all_gather(parts, mine)
        full = torch.zeros((m, fstride), dtype=torch.int64, device="cuda")
        for k in range(world):
            col = 0
            for p in local_panels(k, world, npan):
                nw = (panel_width(p, n, W) + 63) // 64
                full[:, (p * W) // 64:(p * W) // 64 + nw] = parts[k][:, col:col + nw]
                col += nw
        fm = self.f2.DeviceMatrix.from_torch(full, n)
        piv = np.ascontiguousarray(res.pivcols, dtype=np.uint64)
        torch.cuda.synchronize()
        self.f2._check(self.L.f2_pls_compress(fm.handle, res.rank, piv.ctypes.data_as(C.POINTER(C.c_uint64))))
        col = 0
        for p in local_panels(rank, world, npan):
            nw = (panel_width(p, n, W) + 63) // 64
            lt[:, col:col + nw] = full[:, (p * W) // 64:(p * W) // 64 + nw]
            col += nw
        torch.cuda.synchronize()


class TorchComm:
    """broadcast / all_gather over torch.distributed: NCCL for CUDA tensors; with the
    gloo backend (CPU tests, several ranks sharing one GPU) CUDA tensors are staged
    through host memory on the current stream."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.staged = dist.get_backend(group) == "gloo"

    def broadcast(self, buf, root: int):
        if self.staged and buf.is_cuda:
            tmp = buf.cpu()
            self.dist.broadcast(tmp, src=root, group=self.group)
            buf.copy_(tmp)
            return
        self.dist.broadcast(buf, src=root, group=self.group)

    def all_gather(self, parts, mine):
        if self.staged and mine.is_cuda:
            tmp = [p.cpu() for p in parts]
            self.dist.all_gather(tmp, mine.cpu(), group=self.group)
            for p, t in zip(parts, tmp):
                p.copy_(t)
            return
        self.dist.all_gather(parts, mine, group=self.group)
