import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1006_1744_b200 as f2
from oracle_lib import Oracle
o = Oracle()
rng = np.random.default_rng(1)
def rw(m, n):
    w = (n + 63) // 64
    a = rng.integers(0, 2**63, size=(m, w), dtype=np.uint64) * 2 + rng.integers(0, 2, size=(m, w), dtype=np.uint64)
    if n % 64: a[:, -1] &= np.uint64((1 << (n % 64)) - 1)
    return a
for (m, s, n) in [(10, 10, 10), (10, 8, 10), (10, 10, 64), (10, 10, 128), (10, 10, 129), (40, 10, 10), (10, 40, 10), (10, 10, 100)]:
    a, b = rw(m, s), rw(s, n)
    got = f2.mul_m4rm(f2.DeviceMatrix.from_host(a, s), f2.DeviceMatrix.from_host(b, n)).download()
    exp = o.mul(a, s, b, n)
    bad = np.nonzero((got != exp).any(axis=1))[0]
    print((m, s, n), "bad rows", bad[:20], got[bad[:2]] if len(bad) else "", exp[bad[:2]] if len(bad) else "")
