"""Standalone timing of the GEMM behind the Schur update: C (n x n) ^= A (n x K) * B (K x n)
through f2_addmul (tensor-core path for K >= 256; F2_SCHUR_M4RM=1: SMEM table kernel).
usage: python tools/f4_bench.py [n] [K] [reps]"""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = f2.DeviceMatrix(n, n)
c.randomize(0.5, 1)
a = f2.DeviceMatrix(n, K)
a.randomize(0.5, 2)
b = f2.DeviceMatrix(K, n)
b.randomize(0.5, 3)
for _ in range(2):
    f2.addmul(c, a, b)
f2.stats_reset()
f2.stats_enable(True)
for _ in range(reps):
    f2.addmul(c, a, b)
f2.stats_enable(False)
s = f2.stats_get(0)
ms = s["ms"] / s["launches"]
print(f"C {n}x{n} ^= A {n}x{K} * B {K}x{n}: {ms:.3f} ms per call, {2.0 * n * n * K / ms / 1e9:.1f} Tbit-op/s")
