"""Column-sharded PLS (paper_1006_1744_b200/dist.py).

CPU (gloo, world 2 and 3): the schedule, the exchange protocol (buffer layout, lagged
broadcast slices, the stop rule) and the cross-shard compression, with a numpy
per-rank compute standing in for the kernels (test infrastructure), against the
oracle.  GPU: the real kernels (GpuOps, f2_dist_*) -- two processes sharing the box's
GPU over gloo, NCCL at world size 1, and all ranks emulated in one process -- against
the Gaussian oracle: packed matrix (compressed across shards), P, full Q, rank."""
import contextlib
import os
import socket

import numpy as np
import pytest

from oracle_lib import Oracle, ptr

W_TEST = 128


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _case(o, kind, m, n, seed):
    """dense Bernoulli(1/2), rank-deficient X*Y, or fixed-weight sparse rows."""
    if kind == "dense":
        return o.randomize(m, n, 0.5, seed)
    if kind == "xy":
        k = max(1, min(m, n) // 3)
        return o.mul(o.randomize(m, k, 0.5, seed), k, o.randomize(k, n, 0.5, seed + 1), n)
    return o.fixed_weight(m, n, 3, seed)


# ----------------------------------------------------------------------------- CPU ops
def _bit(a, i, j):
    return (int(a[i, j // 64]) >> (j % 64)) & 1


class CpuOps:
    """numpy restatement of f2_dist_factor / f2_dist_step on a local column shard
    (gauss.cpp:33-49 restricted to the panel; trailing columns by the same row
    operations), writing and reading the exchange buffer in the C ABI's layout:
    W/64 words per row, then the header [kb, panel_r, nmoved, col, q[W], P[W], ...].
    Streams are no-ops; the row transpositions travel as the header's P entries."""

    def begin(self, local, m, n, W, npan):
        import torch
        from paper_1006_1744_b200 import dist as D
        self.m, self.W, self.ws = m, W, W // 64
        self.hoff = D.header_offset(m, W)
        self.bufs = [torch.zeros(self.hoff + D.header_words(W), dtype=torch.int64) for _ in range(2)]
        self.r = 0
        self.rk = {}
        self.P = np.arange(m, dtype=np.uint64)
        self.piv = []

    def on_main(self):
        return contextlib.nullcontext()

    on_side = on_main

    def on_comm(self, p):
        return contextlib.nullcontext()

    def main_wait_comm(self):
        pass

    def mark_free(self, p):
        pass

    def slice(self, p, r_lo):
        return self.bufs[p & 1][r_lo * self.ws:]

    def _hdr(self, p):
        return self.bufs[p & 1].numpy().view(np.uint64)[self.hoff:]

    def factor(self, local, p, pw0, width, col):
        a, m, W = local, self.m, self.W
        c0, pos, q, P = pw0 * 64, self.r, [], []
        c = 0
        while pos < m and c < width:
            found = next((i for i in range(pos, m) if _bit(a, i, c0 + c)), -1)
            if found < 0:
                c += 1
                continue
            P.append(found)
            q.append(c)
            if found != pos:
                a[[pos, found]] = a[[found, pos]]
            for i in range(pos + 1, m):  # eliminate below, from c+1 (the L bit stays)
                if _bit(a, i, c0 + c):
                    for j in range(c0 + c + 1, c0 + width):
                        if _bit(a, pos, j):
                            a[i, j // 64] ^= np.uint64(1) << np.uint64(j % 64)
            pos += 1
            c += 1
        kb, r0 = len(q), self.r
        h = self._hdr(p)
        h[:] = 0
        h[0], h[1], h[3] = kb, r0, col
        h[4:4 + kb] = q
        h[4 + W:4 + W + kb] = P
        wv = self.bufs[p & 1].numpy().view(np.uint64)[:self.hoff].reshape(m, self.ws)
        nw = (width + 63) // 64
        wv[r0:, :nw] = a[r0:, pw0:pw0 + nw]
        self.r = r0 + kb

    def step(self, local, p, owner, pw0, width, tw0, lookahead, next_width, next_col):
        a, m, W = local, self.m, self.W
        h = self._hdr(p)
        kb, r = int(h[0]), int(h[1])
        q = [int(x) for x in h[4:4 + kb]]
        P = [int(x) for x in h[4 + W:4 + W + kb]]
        if not owner:
            for t in range(kb):
                if P[t] != r + t:
                    a[[r + t, P[t]]] = a[[P[t], r + t]]
            self.r = r + kb
        if tw0 < a.shape[1]:
            wv = self.bufs[p & 1].numpy().view(np.uint64)[:self.hoff].reshape(m, self.ws)
            for t in range(kb):  # trailing columns: the eliminations in pivot order
                rows = [i for i in range(r + t + 1, m) if (int(wv[i, q[t] // 64]) >> (q[t] % 64)) & 1]
                if rows:
                    a[rows, tw0:] ^= a[r + t, tw0:]
        if lookahead:
            self.factor(local, p + 1, tw0, next_width, next_col)

    def note(self, p):
        h = self._hdr(p)
        kb, r0, col = int(h[0]), int(h[1]), int(h[3])
        self.rk[p] = (kb, r0)
        self.P[r0:r0 + kb] = h[4 + self.W:4 + self.W + kb]
        self.piv.extend(col + int(x) for x in h[4:4 + kb])

    def header_rk(self, p):
        return self.rk[p]

    def finish(self, local):
        return self.r, self.P.copy(), np.asarray(self.piv, dtype=np.uint64)

    def compress_sharded(self, comm, local, m, n, W, rank, world, res):
        import torch
        from paper_1006_1744_b200 import dist as D
        nwk = [(D.local_ncols(k, world, n, W) + 63) // 64 for k in range(world)]
        mine = torch.zeros((m, max(max(nwk), 1)), dtype=torch.int64)
        mine.numpy().view(np.uint64)[:, :local.shape[1]] = local
        parts = [torch.zeros_like(mine) for _ in range(world)]
        comm.all_gather(parts, mine)
        full = D.gather([parts[k].numpy().view(np.uint64)[:, :nwk[k]] for k in range(world)], m, n, W)
        q = np.arange(n, dtype=np.uint64)
        q[:res.rank] = res.pivcols
        Oracle().lib.f2o_compress_columns(ptr(full), m, n, res.rank, ptr(q))
        local[:] = D.split_columns(full, n, rank, world, W)


def _run_rank(rank, world, port, m, n, kind, seed, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1006_1744_b200 import dist as D
    o = Oracle()
    a = _case(o, kind, m, n, seed)
    local = D.split_columns(a, n, rank, world, W_TEST)
    ops, comm = CpuOps(), D.TorchComm()
    res = D.pls_sharded(ops, comm, local, m, n, W_TEST, rank, world)
    D.compress_sharded(ops, comm, local, m, n, W_TEST, rank, world, res)
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), local)
    np.save(os.path.join(out_dir, f"P{rank}.npy"), res.P)
    np.save(os.path.join(out_dir, f"piv{rank}.npy"), res.pivcols)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,kind,seed", [(2, 150, 300, "dense", 1), (2, 300, 200, "xy", 2),
                                                 (2, 97, 333, "sparse", 3), (3, 130, 700, "xy", 4),
                                                 (3, 260, 400, "dense", 5)])
def test_sharded_schedule_gloo(tmp_path, world, m, n, kind, seed):
    import torch.multiprocessing as mp
    from paper_1006_1744_b200 import dist as D
    mp.spawn(_run_rank, args=(world, _free_port(), m, n, kind, seed, str(tmp_path)), nprocs=world, join=True)
    got = D.gather([np.load(tmp_path / f"shard{k}.npy") for k in range(world)], m, n, W_TEST)
    o = Oracle()
    w, p, q, r = o.gauss_pls(_case(o, kind, m, n, seed), n)
    for k in range(world):  # every rank holds the same P and pivot columns
        piv = np.load(tmp_path / f"piv{k}.npy")
        assert piv.size == r and (piv == q[:r]).all()
        assert (np.load(tmp_path / f"P{k}.npy") == p).all()
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


# ----------------------------------------------------------------------------- GPU
def _torch_local(f2, host, ncols):
    import torch
    t = torch.zeros((host.shape[0], f2.DeviceMatrix.stride_for(ncols)), dtype=torch.int64, device="cuda")
    if host.shape[1]:
        t[:, :host.shape[1]] = torch.from_numpy(host.view(np.int64))
    return f2.DeviceMatrix.from_torch(t, ncols)


def _check_against_oracle(oracle, a, m, n, W, got_full, res, q_full, cutoff):
    w, p, q, r = oracle.gauss_pls(a, n)
    assert res.rank == r
    assert (res.P == p).all()
    assert (res.pivcols == q[:r]).all()
    assert (q_full == oracle.recursive_q(m, n, cutoff, q[:r])).all()
    assert (got_full == w).all()


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,W,kind", [(2, 700, 900, 128, "dense"), (3, 1000, 1000, 256, "xy"),
                                              (2, 513, 2000, 1024, "sparse"), (4, 4096, 4096, 512, "dense")])
def test_sharded_gpu_emulated(f2, oracle, world, m, n, W, kind):
    """All ranks' kernels in one process on one stream (the exchange buffer shared, each
    rank's state re-imported from it): multi-shard import/gather/TRSM/Schur paths."""
    from paper_1006_1744_b200 import dist as D
    a = _case(oracle, kind, m, n, m + n + world)
    locals_ = [_torch_local(f2, D.split_columns(a, n, k, world, W), D.local_ncols(k, world, n, W))
               for k in range(world)]
    res = D.pls_sharded_emulated(D.GpuOps(f2), locals_, m, n, W)
    got = D.gather([x.download() for x in locals_], m, n, W)
    g = f2.DeviceMatrix.from_host(got, n)
    f2.compress_columns(g, res.rank, np.concatenate([res.pivcols, np.arange(res.rank, n, dtype=np.uint64)]))
    _check_against_oracle(oracle, a, m, n, W, g.download(), res, D.recursive_q(f2, m, n, 4096, res), 4096)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,W,kind", [(1500, 2300, 512, "dense"), (2048, 2048, 256, "xy"),
                                        (1024, 5000, 1024, "sparse")])
def test_sharded_nccl_world1(f2, oracle, m, n, W, kind):
    """The N > 1 code path of bench.py (pls_sharded with TorchComm over NCCL and GpuOps,
    look-ahead on the side stream) at world size 1 on the box's GPU."""
    import torch
    import torch.distributed as dist
    from paper_1006_1744_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        a = _case(oracle, kind, m, n, 77 + m)
        d = _torch_local(f2, D.split_columns(a, n, 0, 1, W), D.local_ncols(0, 1, n, W))
        ops, comm = D.GpuOps(f2), D.TorchComm()
        res = D.pls_sharded(ops, comm, d, m, n, W, 0, 1)
        D.compress_sharded(ops, comm, d, m, n, W, 0, 1, res)
        got = D.gather([d.download()], m, n, W)
        _check_against_oracle(oracle, a, m, n, W, got, res, D.recursive_q(f2, m, n, 1 << 20, res), 1 << 20)
    finally:
        dist.destroy_process_group()


def _gpu_rank(rank, world, port, m, n, W, kind, out_dir):
    """One rank of the 2-process GPU test: both processes drive the box's GPU, the
    exchange goes through gloo (staged through host memory by TorchComm)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1006_1744_b200 as f2
    from paper_1006_1744_b200 import dist as D
    f2.set_device(0)
    o = Oracle()
    a = _case(o, kind, m, n, 5 + m + n)
    d = _torch_local(f2, D.split_columns(a, n, rank, world, W), D.local_ncols(rank, world, n, W))
    ops, comm = D.GpuOps(f2), D.TorchComm()
    res = D.pls_sharded(ops, comm, d, m, n, W, rank, world)
    D.compress_sharded(ops, comm, d, m, n, W, rank, world, res)
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), d.download())
    np.save(os.path.join(out_dir, f"P{rank}.npy"), res.P)
    np.save(os.path.join(out_dir, f"piv{rank}.npy"), res.pivcols)
    np.save(os.path.join(out_dir, f"Q{rank}.npy"), D.recursive_q(f2, m, n, 4096, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,W,kind", [(1024, 3072, 256, "dense"), (2048, 2048, 512, "xy"),
                                        (512, 4096, 256, "sparse")])
def test_sharded_two_processes(oracle, tmp_path, m, n, W, kind):
    """world_size 2, one process per rank, the product kernels on both (look-ahead on
    the owner of the next panel, async steps, lagged header reads, cross-shard compress)."""
    import torch.multiprocessing as mp
    from paper_1006_1744_b200 import dist as D
    world = 2
    mp.spawn(_gpu_rank, args=(world, _free_port(), m, n, W, kind, str(tmp_path)), nprocs=world, join=True)
    got = D.gather([np.load(tmp_path / f"shard{k}.npy") for k in range(world)], m, n, W)
    a = _case(oracle, kind, m, n, 5 + m + n)
    w, p, q, r = oracle.gauss_pls(a, n)
    qf = oracle.recursive_q(m, n, 4096, q[:r])
    for k in range(world):
        assert (np.load(tmp_path / f"piv{k}.npy") == q[:r]).all()
        assert (np.load(tmp_path / f"P{k}.npy") == p).all()
        assert (np.load(tmp_path / f"Q{k}.npy") == qf).all()
    assert (got == w).all()
