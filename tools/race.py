"""Repeat a dense PLS and count results that differ from the first (or the reference's
digest at 65536): python tools/race.py runs [n]"""
import json
import os
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
want = int(json.load(open("tests/golden/configs.json"))["c3_dense_65536"]["recursive"]["packed_digest"]) if n == 65536 else None
cfg = f2.EliminationConfig(cutoff_bytes=2 << 20)
a0 = f2.DeviceMatrix(n, n)
a0.randomize(0.5, 3)
a = f2.DeviceMatrix(n, n)
bad = []
for i in range(runs):
    a.copy_from(a0)
    r = f2.pls_recursive(a, cfg)
    d = a.digest()
    if want is None:
        want = d
    if d != want or r.rank != n:
        bad.append((i, r.rank, d))
print(f"{os.environ.get('F2_LIB', 'default')} n={n} env={[k for k in os.environ if k.startswith('F2_')]}: {len(bad)} bad of {runs}: {bad[:4]}")
