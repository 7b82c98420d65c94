"""Determinism under interference: a PLS of an m x n dense matrix repeated while another
stream keeps the GPU busy with memory-heavy copies (different timing every run).
python tools/stress.py runs m n"""
import sys

sys.path.insert(0, ".")
import torch

import paper_1006_1744_b200 as f2

runs, m, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
torch.cuda.set_device(0)
cfg = f2.EliminationConfig(cutoff_bytes=2 << 20)
a0 = f2.DeviceMatrix(m, n)
a0.randomize(0.5, 3)
a = f2.DeviceMatrix(m, n)
a.copy_from(a0)
r = f2.pls_recursive(a, cfg)
want = (r.rank, a.digest())
x = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
bg = torch.cuda.Stream()
bad = 0
for i in range(runs):
    with torch.cuda.stream(bg):
        for _ in range(1 + i % 4):
            y.copy_(x)
    a.copy_from(a0)
    r = f2.pls_recursive(a, cfg)
    got = (r.rank, a.digest())
    if got != want:
        bad += 1
        print("run", i, "differs", got, want, flush=True)
torch.cuda.synchronize()
print(f"stress {m}x{n}: {bad} bad of {runs}")
