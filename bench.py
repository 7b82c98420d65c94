#!/usr/bin/env python
"""Benchmark of the B200 GF(2) PLS engine (BASELINE.json: "GF(2) PLS time & effective
Gbit-op/s, 64K^2 dense, 1/2/4/8 B200").

One step = one pls_recursive (pls.hpp:42-47) of the dense 65536x65536 Bernoulli(1/2)
matrix (config 3, cutoff_bytes pinned to 2 MiB), restored from a pristine HBM copy
first.  value = effective bit-ops/s (2 n^3 / 3 per PLS) summed over ranks / device
time (CUDA events on the library stream, max over ranks).  N > 1 (torchrun) runs ONE
65536^2 PLS column-sharded over the ranks with each panel broadcast over NCCL
(paper_1006_1744_b200/dist.py; strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU pls_recursive (oracle/_ref, built from
/root/reference sources) on the box's host cores: every core factors its own seeded
16384^2 sample (the 65536^2 run takes ~6 min on one core), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 65536
SEED = 3
CUTOFF = 2 << 20
BITOPS = 2.0 * N ** 3 / 3.0
METRIC = "GF(2) PLS effective Gbit-op/s (2n^3/3 per decomposition), 64K^2 dense"
UNIT = "Gbit-op/s"
CONFIG = {"workload": "config3: pls_recursive, dense 65536x65536 GF(2), Bernoulli(1/2), seed 3",
          "n": N, "cutoff_bytes": CUTOFF, "panel_bits": 1024,
          "l2": "input 512 MiB > 126 MB L2, restored from an HBM copy every step"}
SAMPLE_N = 16384  # CPU sample size (reference arm / cpu_baseline)
# tcgen05.mma kind::mxf4 128x224x64 with SMEM-resident operands on all 148 SMs (tools/micro/umma_f4,
# profiles/r1_umma_f4_peak.txt): the ceiling of the tensor-core Schur kernel, in fp4 TFLOP/s
F4_MMA_PEAK_TFLOPS = 7500.0
try:
    PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except Exception:
    PEAKS = {}
HBM_GBS = PEAKS.get("hbm_gbs", 6650.0)  # fallback: B200_PROFILING.md


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def reference_rate(steps: int, warmup: int, threads: int, n: int = SAMPLE_N):
    """Reference CPU pls_recursive on `threads` concurrent seeded n x n samples per step.
    Returns (Gbit-op/s aggregate, per-step seconds list)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import RefLib  # reference sources compiled in place (oracle/Makefile)

    R = RefLib()
    inputs = [R.randomize(n, n, 0.5, 1000 + i) for i in range(threads)]
    times = []
    for step in range(warmup + steps):
        out = [None] * threads

        def work(i):
            out[i] = R.pls_recursive(inputs[i], n, CUTOFF)

        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        dt = time.perf_counter() - t0
        if step >= warmup:
            times.append(dt)
    rate = threads * (2.0 * n ** 3 / 3.0) / statistics.median(times) / 1e9
    return rate, times


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libf2ref.so")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libf2ref.so not built"}))
        return 0
    threads = os.cpu_count() or 1
    rate, times = reference_rate(args.steps, args.warmup, threads)
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)", "data": "synthetic (SplitMix64, seeds 1000+i)",
            "config": dict(CONFIG, sample=f"{threads} x pls_recursive {SAMPLE_N}^2 concurrently per step"),
            "impl": "reference",
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{threads} threads, each the reference pls_recursive on its own dense "
                                       f"{SAMPLE_N}^2 matrix (cutoff 2 MiB); the library is single-threaded"},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import numpy as np

    ws, rank, local = dist_env()
    dist = None
    sharded = ws > 1 or args.sharded
    if sharded:
        import torch
        import torch.distributed as dist_mod

        torch.cuda.set_device(local)
        dist_mod.init_process_group("nccl")
        dist = dist_mod

    import paper_1006_1744_b200 as f2

    f2.set_device(local)
    if sharded:
        return run_sharded(args, f2, dist, ws, rank, local)
    cfg = f2.EliminationConfig(cutoff_bytes=CUTOFF)
    a0 = f2.DeviceMatrix(N, N)
    a0.randomize(0.5, SEED + rank)
    a = f2.DeviceMatrix(N, N)

    def barrier():
        if dist:
            import torch
            t = torch.zeros(1, device="cuda")
            dist.all_reduce(t)
            torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step():
        a.copy_from(a0)
        return f2.pls_recursive(a, cfg)

    for _ in range(args.warmup):
        res = step()
    launches = f2.last_graph_kernels() or f2.last_launch_count()

    barrier()
    with Clocks(local) as clk:
        f2.timer_start()
        for _ in range(args.steps):
            res = step()
        ms = f2.timer_stop()
    ms = max_over_ranks(ms)
    ms_per_step = ms / args.steps
    value = ws * args.steps * BITOPS / (ms / 1e3) / 1e9

    # --- dominant kernel roofline: one instrumented (untimed) run.  The stats run times every
    # Schur update with CUDA events on the library stream (the launches of the tensor-core
    # GEMM: A/B operand expansion + k_schur_f4), and reconstructs each launch's work
    # 2 * rows * pivots * trailing columns from the pivot list afterwards.
    f2.stats_reset()
    f2.stats_enable(True)
    step()
    f2.stats_enable(False)
    fam = [f2.stats_get(k) for k in range(4)]
    schur = fam[0]
    total_fam_ms = sum(x["ms"] for x in fam)
    achieved = schur["bitops"] / (schur["ms"] / 1e3) / 1e12 if schur["ms"] else 0.0
    nominal = 9000.0  # fp4 dense, B200_PROFILING.md (MEASURED_PEAKS.json has no fp4 figure)
    roofline = {"kernel": "k_schur_f4 (Schur complement C ^= L21*U12 on tcgen05 kind::mxf4, + operand expansion)",
                "bound": "tensor", "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                "frac": achieved / nominal,
                "peak_source": "nominal fp4 dense 9 PFLOP/s (B200_PROFILING.md table; MEASURED_PEAKS.json has no fp4 "
                               "figure; 4 x its bf16 burst = %.0f)" % (4 * PEAKS.get("bf16_tflops", 0.0)),
                "measured_mma_ceiling": F4_MMA_PEAK_TFLOPS,
                "frac_of_measured_mma_ceiling": achieved / F4_MMA_PEAK_TFLOPS,
                "measured_mma_ceiling_source": "tcgen05.mma kind::mxf4 128x224x64 issue rate with SMEM-resident "
                                               "operands on 148 SMs at 1965 MHz (tools/micro/umma_f4, "
                                               "profiles/r1_umma_f4_peak.txt)",
                "unit_note": "1 GF(2) bit-op = 1 fp4 flop: each AND-count term is one MMA multiply-add",
                "share_of_step": schur["ms"] / total_fam_ms if total_fam_ms else None,
                "launches": schur["launches"], "avg_launch_ms": schur["ms"] / max(schur["launches"], 1),
                "traffic": None}
    prof = os.path.join(ROOT, "profiles", "r1_ncu_schur_f4_config3_raw.json")
    if os.path.exists(prof):
        raw = json.load(open(prof))
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        roofline["traffic"] = sum(float(raw[k][0]) * scale.get(raw[k][1], 1.0)
                                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        roofline["traffic_note"] = ("dram read+write bytes of the first wide k_schur_f4 launch of config 3 "
                                    "(ncu --set full, profiles/r1_ncu_schur_f4_config3_raw.json); its algorithmic "
                                    "bytes (C read+write once) are %.4g" % (64512 * 63488 / 8 * 2))

    # --- MMPF table-apply (k_mmpf_apply, K <= 64) over a 1 GiB trailing matrix: the HBM-bound
    # kernel of the flat MMPF; K = 8 is the paper's single 2^8 table, K = 64 the engine's MMPF panel
    table_apply = {}
    if rank == 0:
        rows, cols = 65536, 131072
        c = f2.DeviceMatrix(rows, cols)
        c.randomize(0.5, 11)
        for kbits in (8, 64):
            am = f2.DeviceMatrix(rows, kbits)
            am.randomize(0.5, 12)
            bm = f2.DeviceMatrix(kbits, cols)
            bm.randomize(0.5, 13)
            for _ in range(3):
                f2.addmul(c, am, bm)
            f2.stats_reset()
            f2.stats_enable(True)
            for _ in range(5):
                f2.addmul(c, am, bm)
            f2.stats_enable(False)
            st = f2.stats_get(0)
            gbs = st["bytes"] / (st["ms"] / 1e3) / 1e9
            table_apply[f"k{kbits}"] = {"GB_s": gbs, "frac_of_measured_hbm": gbs / HBM_GBS,
                                        "ms_per_launch": st["ms"] / st["launches"],
                                        "bytes_per_launch": st["bytes"] / st["launches"],
                                        "shape": f"C {rows}x{cols} ^= A {rows}x{kbits} * B {kbits}x{cols}"}
            del am, bm
        del c

    # --- e2e through the host-buffer C-ABI call (pinned buffers, copies inside the timed region)
    e2e = None
    if rank == 0 or True:
        words = (N + 63) // 64
        h0 = f2.pinned_empty((N, words))
        a0.download(h0)
        h = f2.pinned_empty((N, words))
        e2e_steps = max(1, min(args.steps, 3))
        tot = 0.0
        for i in range(e2e_steps + 1):
            np.copyto(h, h0)
            f2.timer_start()
            f2.pls_recursive_host(h, N, cfg)
            dt = f2.timer_stop()
            if i > 0:
                tot += dt
        tot = max_over_ranks(tot)
        e2e = {"value": ws * e2e_steps * BITOPS / (tot / 1e3) / 1e9, "unit": UNIT,
               "ms_per_step": tot / e2e_steps, "h2d_bytes_per_step": N * words * 8,
               "d2h_bytes_per_step": N * words * 8 + 8 * 2 * N, "steps": e2e_steps,
               "call": "f2_pls_recursive_host (upload, decompose, download P/Q/L\\S)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            rate, times = reference_rate(1, 0, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{threads} threads, each the reference pls_recursive on its own dense {SAMPLE_N}^2 "
                             f"matrix (cutoff 2 MiB), one step, {times[0]:.1f} s wall"}
        except Exception as e:  # the reference build is test infrastructure; report, do not fail
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)",
                "data": "synthetic (BitMatrix::randomize SplitMix64 stream, seed 3 + rank, generated on device)",
                "config": dict(CONFIG, parallelism=f"replicas x{ws}"),
                "rank": res.rank, "clocks": clk.summary(), "e2e": e2e, "roofline": roofline,
                "table_apply_hbm": table_apply, "cpu_baseline": cpu,
                "gpu_launches": launches * args.steps,
                "gpu_launches_note": "kernel nodes of the replayed CUDA graph per PLS x steps",
                "kernel_families_ms": {k: fam[i]["ms"] for i, k in enumerate(["schur", "panel", "trsm", "other"])}}
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def run_sharded(args, f2, dist, ws, rank, local):
    """N > 1: one 65536^2 PLS column-sharded over the ranks (paper_1006_1744_b200/dist.py),
    panel data broadcast with NCCL; strong scaling (total work fixed)."""
    import numpy as np
    import torch

    from paper_1006_1744_b200 import dist as D

    W = 1024
    full = f2.DeviceMatrix(N, N)
    full.randomize(0.5, SEED)
    host = full.download()
    del full
    shard = D.split_columns(host, N, rank, ws, W)
    ncols = D.local_ncols(rank, ws, N, W)
    a0 = f2.DeviceMatrix.from_host(shard, ncols)
    a = f2.DeviceMatrix(N, ncols)
    del host, shard
    ops, comm = D.GpuOps(f2), D.TorchComm()

    def step():
        a.copy_from(a0)
        return D.pls_sharded(ops, comm, a, N, N, W, rank, ws)

    for _ in range(args.warmup):
        res = step()
    t = torch.zeros(1, device="cuda")
    dist.all_reduce(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            res = step()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    if rank == 0:
        line = {"metric": METRIC, "value": args.steps * BITOPS / (ms / 1e3) / 1e9, "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)",
                "data": "synthetic (BitMatrix::randomize SplitMix64 stream, seed 3)",
                "config": dict(CONFIG, parallelism=f"column-sharded x{ws} (block-cyclic {W}-bit panels, NCCL broadcast)"),
                "rank": res.rank, "clocks": clk.summary(), "e2e": None, "roofline": None, "cpu_baseline": None,
                "gpu_launches": None}
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--sharded", action="store_true",
                    help="the column-sharded NCCL schedule even at one rank (exercises the N > 1 path)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
