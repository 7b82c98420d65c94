"""Column-sharded PLS (paper_1006_1744_b200/dist.py).

CPU (gloo, world_size 2): the schedule and the exchange protocol, with a numpy
per-rank compute standing in for the kernels (test infrastructure), against the
oracle.  GPU: the real kernels with all ranks emulated on one device, against the
single-GPU engine and the oracle (bit-exact packed matrix, P, pivot columns)."""
import os

import numpy as np
import pytest

from oracle_lib import Oracle, words

W_TEST = 128


# ----------------------------------------------------------------------------- CPU ops
def _bit(a, i, j):
    return (int(a[i, j // 64]) >> (j % 64)) & 1


class CpuOps:
    """numpy restatement of factor_panel / apply_panel on a local column shard
    (gauss.cpp:33-49 restricted to the panel; trailing columns by the same row
    operations).  Transpositions travel in the header's P entries."""
    kmax_moved = 8192

    def exchange_buffers(self, m, W):
        import torch
        self.W = W
        hw = 4 + 2 * W + 2 * self.kmax_moved
        self.hdr = torch.zeros(hw, dtype=torch.int64)
        self.words = torch.zeros(m * (W // 64), dtype=torch.int64)
        return self.hdr, self.words

    def begin(self, local):
        pass

    def read_header(self, hdr):
        return hdr.numpy().view(np.uint64)

    def factor_panel(self, local, pw0, width, r, panel_col, hdr, words):
        a = local
        m = a.shape[0]
        c0 = pw0 * 64
        pos, q, P = r, [], []
        col = 0
        while pos < m and col < width:
            found = -1
            for i in range(pos, m):
                if _bit(a, i, c0 + col):
                    found = i
                    break
            if found < 0:
                col += 1
                continue
            P.append(found)
            q.append(col)
            if found != pos:
                tmp = a[pos].copy()
                a[pos] = a[found]
                a[found] = tmp
            # eliminate below within the panel, from col+1 (the L bit stays)
            lo = c0 + col + 1
            for i in range(pos + 1, m):
                if _bit(a, i, c0 + col):
                    for j in range(lo, c0 + width):
                        if _bit(a, pos, j):
                            a[i, j // 64] ^= np.uint64(1) << np.uint64(j % 64)
            pos += 1
            col += 1
        kb = len(q)
        h = hdr.numpy().view(np.uint64)
        h[:] = 0
        h[0], h[1] = kb, r
        W = self.W
        h[4:4 + kb] = q
        h[4 + W + 2 * self.kmax_moved:4 + W + 2 * self.kmax_moved + kb] = P
        wv = words.numpy().view(np.uint64).reshape(m, W // 64)
        nw = (width + 63) // 64
        wv[r:, :nw] = a[r:, pw0:pw0 + nw]
        return kb

    def apply_panel(self, local, tw0, width, owner, hdr, words):
        a = local
        m = a.shape[0]
        h = hdr.numpy().view(np.uint64)
        kb, r = int(h[0]), int(h[1])
        W = self.W
        q = [int(x) for x in h[4:4 + kb]]
        P = [int(x) for x in h[4 + W + 2 * self.kmax_moved:4 + W + 2 * self.kmax_moved + kb]]
        if not owner:
            for t in range(kb):
                if P[t] != r + t:
                    tmp = a[r + t].copy()
                    a[r + t] = a[P[t]]
                    a[P[t]] = tmp
        if tw0 >= a.shape[1]:
            return
        wv = words.numpy().view(np.uint64).reshape(m, W // 64)
        for t in range(kb):  # trailing columns: the eliminations in pivot order
            qt = q[t]
            rows = [i for i in range(r + t + 1, m) if (int(wv[i, qt // 64]) >> (qt % 64)) & 1]
            if rows:
                a[rows, tw0:] ^= a[r + t, tw0:]


def _run_rank(rank, world, port, m, n, seed, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_1006_1744_b200 import dist as D
    o = Oracle()
    a = o.randomize(m, n, 0.5 if seed % 2 else 0.1, seed)
    local = D.split_columns(a, n, rank, world, W_TEST)
    res = D.pls_sharded(CpuOps(), D.TorchComm(), local, m, n, W_TEST, rank, world)
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), local)
    if rank == 0:
        np.save(os.path.join(out_dir, "P.npy"), res.P)
        np.save(os.path.join(out_dir, "piv.npy"), res.pivcols)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,seed", [(150, 300, 1), (300, 200, 2), (97, 333, 3)])
def test_sharded_schedule_gloo_world2(tmp_path, m, n, seed):
    import torch.multiprocessing as mp
    from paper_1006_1744_b200 import dist as D
    port = 29500 + seed * 7 + os.getpid() % 100
    mp.spawn(_run_rank, args=(2, port, m, n, seed, str(tmp_path)), nprocs=2, join=True)
    shards = [np.load(tmp_path / f"shard{k}.npy") for k in range(2)]
    got = D.gather(shards, m, n, W_TEST)
    o = Oracle()
    a = o.randomize(m, n, 0.5 if seed % 2 else 0.1, seed)
    w, p, q, r = o.gauss_pls(a, n)
    piv = np.load(tmp_path / "piv.npy")
    assert piv.size == r and (piv == q[:r]).all()
    assert (np.load(tmp_path / "P.npy") == p).all()
    # the sharded path leaves L at the pivot columns (uncompressed); compress like the engine
    import ctypes
    from oracle_lib import ptr
    o.lib.f2o_compress_columns(ptr(got), m, n, r, ptr(np.ascontiguousarray(q)))
    assert (got == w).all()


def test_shard_layout_roundtrip():
    from paper_1006_1744_b200 import dist as D
    o = Oracle()
    m, n, W = 40, 700, 128
    a = o.randomize(m, n, 0.5, 9)
    for world in (1, 2, 3, 4):
        shards = [D.split_columns(a, n, k, world, W) for k in range(world)]
        assert sum(D.local_ncols(k, world, n, W) for k in range(world)) == n
        assert (D.gather(shards, m, n, W) == a).all()
        for p in range((n + W - 1) // W):
            k = D.owner_of(p, world)
            assert D.local_word0(p, k, world, W) == D.first_trailing_word(p, k, world, W) - W // 64


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,W", [(2, 700, 900, 128), (3, 1000, 1000, 256), (2, 513, 2000, 1024),
                                         (4, 4096, 4096, 512)])
def test_sharded_gpu_emulated(f2, oracle, world, m, n, W):
    from paper_1006_1744_b200 import dist as D
    a = oracle.randomize(m, n, 0.5, m + n + world)
    locals_ = [f2.DeviceMatrix.from_host(D.split_columns(a, n, k, world, W), D.local_ncols(k, world, n, W))
               for k in range(world)]
    res = D.pls_sharded_emulated(D.GpuOps(f2), locals_, m, n, W)
    got = D.gather([x.download() for x in locals_], m, n, W)
    w, p, q, r = oracle.gauss_pls(a, n)
    assert res.rank == r and (res.P == p).all() and (res.pivcols == q[:r]).all()
    g = f2.DeviceMatrix.from_host(got, n)
    f2.load_library().f2_pls_compress.argtypes = [__import__("ctypes").c_void_p, __import__("ctypes").c_uint64,
                                                  __import__("ctypes").POINTER(__import__("ctypes").c_uint64)]
    pc = np.ascontiguousarray(res.pivcols)
    f2._check(f2.load_library().f2_pls_compress(g.handle, res.rank, pc.ctypes.data_as(
        __import__("ctypes").POINTER(__import__("ctypes").c_uint64))))
    assert (g.download() == w).all()


@pytest.mark.gpu
def test_sharded_nccl_world1(f2, oracle):
    """The N > 1 code path of bench.py (pls_sharded with TorchComm over NCCL and GpuOps)
    at world size 1, one process on the box's GPU: the real NCCL broadcast of the header
    and panel words, checked against the Gaussian oracle."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_1006_1744_b200 import dist as D
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        m, n, W = 1500, 2300, 512
        a = oracle.randomize(m, n, 0.5, 77)
        d = f2.DeviceMatrix.from_host(D.split_columns(a, n, 0, 1, W), D.local_ncols(0, 1, n, W))
        res = D.pls_sharded(D.GpuOps(f2), D.TorchComm(), d, m, n, W, 0, 1)
        w, p, q, r = oracle.gauss_pls(a, n)
        assert res.rank == r and (res.P == p).all() and (res.pivcols == q[:r]).all()
        got = D.gather([d.download()], m, n, W)
        g = f2.DeviceMatrix.from_host(got, n)
        import ctypes as C
        L = f2.load_library()
        L.f2_pls_compress.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        pc = np.ascontiguousarray(res.pivcols)
        f2._check(L.f2_pls_compress(g.handle, res.rank, pc.ctypes.data_as(C.POINTER(C.c_uint64))))
        assert (g.download() == w).all()
    finally:
        dist.destroy_process_group()
