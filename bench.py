#!/usr/bin/env python
"""Benchmark of the B200 GF(2) PLS engine (BASELINE.json: "GF(2) PLS time & effective
Gbit-op/s, 64K^2 dense, 1/2/4/8 B200").

One step = one pls_recursive (pls.hpp:42-47) of the dense 65536x65536 Bernoulli(1/2)
matrix (config 3, cutoff_bytes pinned to 2 MiB), restored from a pristine HBM copy
first.  value = effective bit-ops/s (2 n^3 / 3 per PLS) / device time (CUDA events).
N > 1 runs ONE 65536^2 PLS column-sharded over the ranks (paper_1006_1744_b200/dist.py:
block-cyclic 1024-column panels, each panel's header and L block broadcast over NCCL,
look-ahead on the owner of the next panel; strong scaling), timed as the max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1).

--impl reference times the reference's own CPU pls_recursive (oracle/_ref, the
reference sources compiled as shipped) on the box's host cores, rank 0 only.  The
reference is single-threaded and one 65536^2 decomposition takes ~200 s on one core
(profiles/r2_reference_configs_cpu.json), so each step is a bounded sample of the same
workload: every host core factors its own seeded 16384^2 matrix with the same cutoff
(its per-core rate is ~1.9x the 65536^2 rate, so the ratio against it is conservative).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
W_SHARD = 1024
BITOPS = 2.0 * N ** 3 / 3.0
METRIC = "GF(2) PLS effective Gbit-op/s (2n^3/3 per decomposition), 64K^2 dense"
UNIT = "Gbit-op/s"
SAMPLE_N = 16384  # CPU sample size (reference arm / cpu_baseline)
# tcgen05.mma kind::mxf4 128x224x64 with SMEM-resident operands on all 148 SMs, issued without
# draining the pipe (tools/micro/umma_f4_pair, profiles/r2_umma_f4_pair_peak.txt): the ceiling of
# the tensor-core Schur kernel's data path, in fp4 TFLOP/s
F4_MMA_PEAK_TFLOPS = 8880.0
F4_NOMINAL_TFLOPS = 9000.0  # fp4 dense, B200_PROFILING.md (MEASURED_PEAKS.json has no fp4 figure)
try:
    PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except Exception:
    PEAKS = {}
HBM_GBS = PEAKS.get("hbm_gbs", 6650.0)  # fallback: B200_PROFILING.md
GOLDEN = os.path.join(ROOT, "tests", "golden", "configs.json")  # digests of the reference's outputs
REF_CONFIGS = os.path.join(ROOT, "profiles", "r2_reference_configs_cpu.json")


def config_for(ws: int) -> dict:
    """The workload of this line; the reference arm prints the same dict for the same N."""
    return {"workload": "config3: pls_recursive, dense 65536x65536 GF(2), Bernoulli(1/2), seed 3",
            "n": N, "cutoff_bytes": CUTOFF, "panel_bits": 1024,
            "l2": "input 512 MiB > 126 MB L2, restored from an HBM copy every step",
            "parallelism": "single GPU" if ws == 1 else
            f"column-sharded x{ws} (block-cyclic {W_SHARD}-bit panels, NCCL broadcast of each panel)"}


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


def golden():
    try:
        return json.load(open(GOLDEN))
    except Exception:
        return {}


# --------------------------------------------------------------------------- reference arm
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


def reference_sample(threads: int) -> str:
    return (f"{threads} threads, each the reference pls_recursive on its own dense {SAMPLE_N}^2 matrix "
            f"(cutoff 2 MiB, seeds 1000+i) per step; the library is single-threaded and one 65536^2 run "
            f"takes ~200 s on one core, so the sample is a bounded slice of the config-3 workload")


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
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)",
            "data": "synthetic (SplitMix64, seeds 1000+i)", "config": config_for(ws), "impl": "reference",
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": reference_sample(threads)},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- helpers
def barrier_and_max(dist):
    import torch

    def barrier():
        if dist:
            t = torch.zeros(1, device="cuda")
            dist.all_reduce(t)
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    return barrier, max_over_ranks


def schur_roofline(fam0, total_ms, note):
    achieved = fam0["bitops"] / (fam0["ms"] / 1e3) / 1e12 if fam0["ms"] else 0.0
    r = {"kernel": "k_schur_f4 (Schur complement C ^= L21*U12 on tcgen05 kind::mxf4, + operand expansion)",
         "bound": "tensor", "achieved": achieved, "peak": F4_NOMINAL_TFLOPS, "unit": "TFLOP/s",
         "frac": achieved / F4_NOMINAL_TFLOPS,
         "peak_source": "nominal fp4 dense 9 PFLOP/s (B200_PROFILING.md table; MEASURED_PEAKS.json has no fp4 "
                        "figure; 4 x its bf16 burst = %.0f)" % (4 * PEAKS.get("bf16_tflops", 0.0)),
         "measured_mma_ceiling": F4_MMA_PEAK_TFLOPS,
         "frac_of_measured_mma_ceiling": achieved / F4_MMA_PEAK_TFLOPS,
         "measured_mma_ceiling_source": "tcgen05.mma kind::mxf4 128x224x64 back to back with SMEM-resident operands "
                                        "on 148 SMs at 1965 MHz, no pipe drain (tools/micro/umma_f4_pair, "
                                        "profiles/r2_umma_f4_pair_peak.txt; the CTA-pair form measures the same)",
         "unit_note": "1 GF(2) bit-op = 1 fp4 flop: each AND-count term is one MMA multiply-add",
         "per_unit": "2 * rows * pivots * columns bit-ops per Schur launch (rows below the panel's pivots, the "
                     "panel's pivots, the trailing columns), summed from the pivot list",
         "share_of_step": fam0["ms"] / total_ms if total_ms else None,
         "launches": fam0["launches"], "avg_launch_ms": fam0["ms"] / max(fam0["launches"], 1),
         "timing": note, "traffic": None}
    prof = os.path.join(ROOT, "profiles", "r2_ncu_schur_f4_config3_raw.json")
    if os.path.exists(prof):
        raw = json.load(open(prof))
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        r["traffic"] = sum(float(raw[k][0]) * scale.get(raw[k][1], 1.0)
                           for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        r["traffic_note"] = ("dram read+write bytes of the first wide k_schur_f4 launch of config 3 (ncu --set full, "
                             "profiles/r2_ncu_schur_f4_config3_raw.json); its algorithmic bytes (C read+write once) "
                             "are %.4g" % (64512 * 63488 / 8 * 2))
        clk = float(raw.get("sm__cycles_elapsed.avg.per_second", ["0"])[0] or 0)
        if clk:
            r["sustained_clock_ghz"] = clk
            r["frac_of_mma_ceiling_at_sustained_clock"] = (
                8.39e12 / (float(raw["gpu__time_duration.sum"][0]) * 1e-3) / 1e12 / (F4_MMA_PEAK_TFLOPS * clk / 1.965))
            r["clock_note"] = ("under sustained fp4 load the kernel runs power-capped (ncu: %.2f GHz); at that clock the "
                               "launch profiled reaches the fraction above of the MMA-only ceiling" % clk)
    return r


def table_apply_hbm(f2):
    """MMPF table-apply (k_mmpf_apply, K <= 64) over a 1 GiB trailing matrix: the HBM-bound
    kernel of the flat MMPF; K = 8 is the paper's single 2^8 table, K = 64 the engine's MMPF panel."""
    out = {}
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
        out[f"k{kbits}"] = {"GB_s": gbs, "frac_of_measured_hbm": gbs / HBM_GBS,
                            "ms_per_launch": st["ms"] / st["launches"], "bytes_per_launch": st["bytes"] / st["launches"],
                            "per_unit": "rows x (2 x 8 x trailing words + 8 x coefficient words) + B rows",
                            "shape": f"C {rows}x{cols} ^= A {rows}x{kbits} * B {kbits}x{cols}"}
    return out


def per_config(f2, np):
    """Device and end-to-end time of configs 1, 2, 4 and 5 (BASELINE.json) through the
    paths SURVEY.md §8d lists, each checked against the reference's digests
    (tests/golden/configs.json), beside the reference's single-core time of the same
    config on this kind of host (profiles/r2_reference_configs_cpu.json)."""
    gold = golden()
    try:
        ref = json.load(open(REF_CONFIGS))["configs"]
    except Exception:
        ref = {}
    out = {}
    for name in ("c1_dense_4096", "c2_dense_16384", "c4_xy_32768", "c5_sparse_16384x131072"):
        g = gold.get(name)
        if not g:
            continue
        m, n = g["m"], g["n"]
        if g["kind"] == "dense":
            a0 = f2.DeviceMatrix(m, n)
            a0.randomize(0.5, g["seed"])
        elif g["kind"] == "xy":
            x = f2.DeviceMatrix(m, g["inner"])
            x.randomize(0.5, g["seed_x"])
            y = f2.DeviceMatrix(g["inner"], n)
            y.randomize(0.5, g["seed_y"])
            a0 = f2.mul_m4rm(x, y)
            del x, y
        else:
            a0 = f2.DeviceMatrix(m, n)
            a0.fixed_weight(g["weight"], g["seed"])
        entry = {"m": m, "n": n, "input_matches_reference": a0.digest() == int(g["input_digest"])}
        bitops = 2.0 * n ** 3 / 3.0 if m == n else m * m * n - m ** 3 / 3.0
        entry["bitops"] = bitops
        cfg = f2.EliminationConfig(cutoff_bytes=int(g["cutoff_bytes"]))
        a = f2.DeviceMatrix(m, n)
        host0 = a0.download(f2.pinned_empty((m, (n + 63) // 64)))
        host = f2.pinned_empty(host0.shape)
        for path in g["paths"]:
            run = (lambda: f2.mmpf_pls(a)) if path == "mmpf" else (lambda: f2.pls_recursive(a, cfg))
            reps = 5 if m * n <= (1 << 28) else 3
            times = []
            for i in range(reps + 1):
                a.copy_from(a0)
                f2.timer_start()
                res = run()
                dt = f2.timer_stop()
                if i:
                    times.append(dt)
            ok = (res.rank == g[path]["rank"] and a.digest() == int(g[path]["packed_digest"]))
            host_fn = (lambda: f2.mmpf_pls_host(host, n)) if path == "mmpf" else \
                (lambda: f2.pls_recursive_host(host, n, cfg))
            et = []
            for i in range(reps + 1):
                np.copyto(host, host0)
                f2.timer_start()
                host_fn()
                dt = f2.timer_stop()
                if i:
                    et.append(dt)
            dev_ms, e2e_ms = statistics.median(times), statistics.median(et)
            r1 = ref.get(name, {}).get(path if path == "mmpf" else "recursive", {})
            e = {"device_ms": dev_ms, "e2e_ms": e2e_ms, "gbitops_device": bitops / dev_ms / 1e6,
                 "gbitops_e2e": bitops / e2e_ms / 1e6, "rank": res.rank, "matches_reference_digests": ok,
                 "e2e_h2d_bytes": host0.nbytes, "e2e_d2h_bytes": host0.nbytes + 8 * (m + n)}
            if r1.get("seconds"):
                e["reference_1core_s"] = r1["seconds"]
                e["speedup_e2e_vs_reference_1core"] = 1e3 * r1["seconds"] / e2e_ms
            entry[path] = e
        out[name] = entry
        del a, a0
    return out


# --------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np

    ws, rank, local = dist_env()
    if ws > 1 or args.sharded:
        return run_sharded(args, ws, rank, local)
    import paper_1006_1744_b200 as f2

    f2.set_device(local)
    cfg = f2.EliminationConfig(cutoff_bytes=CUTOFF)
    a0 = f2.DeviceMatrix(N, N)
    a0.randomize(0.5, SEED)
    a = f2.DeviceMatrix(N, N)

    def step():
        a.copy_from(a0)
        return f2.pls_recursive(a, cfg)

    for _ in range(args.warmup):
        res = step()
    launches = f2.last_graph_kernels() or f2.last_launch_count()
    with Clocks(local) as clk:
        f2.timer_start()
        for _ in range(args.steps):
            res = step()
        ms = f2.timer_stop()
    ms_per_step = ms / args.steps
    value = args.steps * BITOPS / (ms / 1e3) / 1e9
    g3 = golden().get("c3_dense_65536", {}).get("recursive", {})
    check = {"rank": res.rank, "packed_matches_reference": a.digest() == int(g3.get("packed_digest", -1))}

    # dominant kernel roofline: one instrumented (untimed) run.  The stats run times every
    # Schur update with CUDA events on the library stream (the tensor-core GEMM launches:
    # A/B operand expansion + k_schur_f4) and reconstructs each launch's work
    # 2 * rows * pivots * trailing columns from the pivot list afterwards.
    f2.stats_reset()
    f2.stats_enable(True)
    step()
    f2.stats_enable(False)
    fam = [f2.stats_get(k) for k in range(4)]
    roofline = schur_roofline(fam[0], sum(x["ms"] for x in fam), "stats run: launches serialised, no look-ahead")

    table_apply = table_apply_hbm(f2)

    # e2e through the host-buffer C-ABI call (pinned buffers, copies inside the timed region)
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
    chk = f2.DeviceMatrix.from_host(h, N)
    check["e2e_packed_matches_reference"] = chk.digest() == int(g3.get("packed_digest", -1))
    del chk
    e2e = {"value": e2e_steps * BITOPS / (tot / 1e3) / 1e9, "unit": UNIT, "ms_per_step": tot / e2e_steps,
           "h2d_bytes_per_step": N * words * 8, "d2h_bytes_per_step": N * words * 8 + 8 * 2 * N, "steps": e2e_steps,
           "call": "f2_pls_recursive_host (upload, decompose, download P/Q/L\\S)"}

    configs = {} if args.no_configs else per_config(f2, np)

    cpu = None
    if not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            rate, times = reference_rate(1, 0, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": reference_sample(threads) + f"; one step, {times[0]:.1f} s wall"}
            c2 = configs.get("c2_dense_16384", {}).get("recursive")
            if c2:  # same size as the sample: a same-config GPU/CPU comparison
                cpu["config2_same_size"] = {"gpu_device_gbitops": c2["gbitops_device"],
                                            "gpu_e2e_gbitops": c2["gbitops_e2e"],
                                            "ratio_e2e_vs_all_cores": c2["gbitops_e2e"] / rate}
        except Exception as e:  # the reference build is test infrastructure; report, do not fail
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    try:
        r3 = json.load(open(REF_CONFIGS))["configs"]["c3_dense_65536"]["recursive"]["seconds"]
        ref_full = {"seconds_1core": r3, "gbitops_1core": BITOPS / r3 / 1e9,
                    "speedup_e2e": r3 * 1e3 / e2e["ms_per_step"],
                    "source": "profiles/r2_reference_configs_cpu.json (reference pls_recursive, this config, one "
                              "core of the GPU box's host, digests equal to tests/golden)"}
    except Exception:
        ref_full = None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)",
            "data": "synthetic (BitMatrix::randomize SplitMix64 stream, seed 3, generated on device)",
            "config": config_for(ws), "check": check, "clocks": clk.summary(), "e2e": e2e, "roofline": roofline,
            "table_apply_hbm": table_apply, "cpu_baseline": cpu, "reference_config3_full": ref_full,
            "configs": configs, "gpu_launches": launches * args.steps,
            "gpu_launches_note": "kernel nodes of the replayed CUDA graph per PLS x steps",
            "kernel_families_ms": {k: fam[i]["ms"] for i, k in enumerate(["schur", "panel", "trsm", "other"])}}
    print(json.dumps(line))
    return 0


def run_sharded(args, ws, rank, local):
    """N > 1: one 65536^2 PLS column-sharded over the ranks (paper_1006_1744_b200/dist.py);
    strong scaling (total work fixed), device time = max over ranks of CUDA events bracketing
    the step on every rank."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1006_1744_b200 as f2
    from paper_1006_1744_b200 import dist as D

    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", local))
    f2.set_device(local)
    W = W_SHARD
    npan = N // W
    ncols = D.local_ncols(rank, ws, N, W)
    lstride = f2.DeviceMatrix.stride_for(ncols)
    full_t = torch.zeros((N, f2.DeviceMatrix.stride_for(N)), dtype=torch.int64, device="cuda")
    f2.DeviceMatrix.from_torch(full_t, N).randomize(0.5, SEED)
    cols = [c for p in D.local_panels(rank, ws, npan) for c in range(p * W // 64, (p + 1) * W // 64)]
    a0_t = torch.zeros((N, lstride), dtype=torch.int64, device="cuda")
    a0_t[:, :len(cols)] = full_t[:, cols]
    del full_t
    a_t = torch.zeros_like(a0_t)
    a = f2.DeviceMatrix.from_torch(a_t, ncols)
    # from N = 2 on the per-rank trailing update no longer hides the panel kernel, which is then
    # the critical path from the first panel: give it the late schedule's CTA count throughout
    ops, comm = D.GpuOps(f2, side_ctas=48 if ws > 1 else 0), D.TorchComm()
    barrier, max_over_ranks = barrier_and_max(dist)

    def step():
        a_t.copy_(a0_t)
        return D.pls_sharded(ops, comm, a, N, N, W, rank, ws)

    for _ in range(args.warmup):
        res = step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        e1.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1))
    value = args.steps * BITOPS / (ms / 1e3) / 1e9

    # Schur roofline inside the timed schedule (events around each Schur launch on this rank's
    # main stream; the look-ahead stays on), summed over ranks
    f2.stats_reset()
    f2.stats_enable(True)
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    step()
    t1.record()
    t1.synchronize()
    f2.stats_enable(False)
    s0 = f2.stats_get(0)
    tot = torch.tensor([s0["bitops"], s0["ms"], float(s0["launches"])], dtype=torch.float64, device="cuda")
    dist.all_reduce(tot)
    fam0 = {"bitops": tot[0].item(), "ms": tot[1].item(), "launches": int(tot[2].item())}
    roofline = schur_roofline(fam0, ws * t0.elapsed_time(t1),
                              f"stats run of the sharded schedule (look-ahead on), Schur time summed over {ws} ranks")

    # e2e: every rank uploads its column shard from pinned host memory, runs, downloads it
    lw = (ncols + 63) // 64
    hl0 = f2.pinned_empty((N, lw))
    a_t.copy_(a0_t)
    torch.cuda.synchronize()
    a.download(hl0)
    hl = f2.pinned_empty((N, lw))
    e2e_steps = max(1, min(args.steps, 3))
    tot_ms = 0.0
    for i in range(e2e_steps + 1):
        np.copyto(hl, hl0)
        barrier()
        t0.record()
        a.upload(hl)
        res = D.pls_sharded(ops, comm, a, N, N, W, rank, ws)
        D.compress_sharded(ops, comm, a, N, N, W, rank, ws, res)
        a.download(hl)
        q = D.recursive_q(f2, N, N, CUTOFF, res)
        t1.record()
        t1.synchronize()
        if i:
            tot_ms += t0.elapsed_time(t1)
    tot_ms = max_over_ranks(tot_ms)
    e2e = {"value": e2e_steps * BITOPS / (tot_ms / 1e3) / 1e9, "unit": UNIT, "ms_per_step": tot_ms / e2e_steps,
           "h2d_bytes_per_step": N * (N // 64) * 8, "d2h_bytes_per_step": N * (N // 64) * 8 + 8 * 2 * N,
           "steps": e2e_steps, "call": "per rank: upload of the column shard from pinned memory, dist.pls_sharded, "
                                       "compress_sharded, download of the shard and P/Q"}

    # correctness of the timed path at full size: the gathered packed matrix against the
    # reference's digest (outside every timed region)
    g3 = golden().get("c3_dense_65536", {}).get("recursive", {})
    parts = [torch.empty_like(a0_t) for _ in range(ws)]
    dist.all_gather(parts, a_t)
    check = {"rank": res.rank}
    if rank == 0:
        full = torch.zeros((N, f2.DeviceMatrix.stride_for(N)), dtype=torch.int64, device="cuda")
        for k in range(ws):
            kc = [c for p in D.local_panels(k, ws, npan) for c in range(p * W // 64, (p + 1) * W // 64)]
            full[:, kc] = parts[k][:, :len(kc)]
        fm = f2.DeviceMatrix.from_torch(full, N)
        check["packed_matches_reference"] = fm.digest() == int(g3.get("packed_digest", -1))
        check["q_is_identity"] = bool((q == np.arange(N, dtype=np.uint64)).all())
        del fm, full
    del parts

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)",
                "data": "synthetic (BitMatrix::randomize SplitMix64 stream, seed 3, generated on device)",
                "config": config_for(ws), "check": check, "clocks": clk.summary(), "e2e": e2e, "roofline": roofline,
                "cpu_baseline": None, "cpu_baseline_note": "timed at N = 1 only (rank 0), as the bench contract asks",
                "gpu_launches": None, "path": "dist.pls_sharded (f2_dist_* C ABI, NCCL)"}
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config timings of configs 1, 2, 4, 5")
    ap.add_argument("--sharded", action="store_true",
                    help="the column-sharded NCCL schedule even at one rank (exercises the N > 1 path)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={ws}"}), file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
