"""Config-3 device time only (A/B of schedule switches): python tools/t3.py [n] [steps]."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = f2.EliminationConfig(cutoff_bytes=2 << 20)
a0 = f2.DeviceMatrix(n, n)
a0.randomize(0.5, 3)
a = f2.DeviceMatrix(n, n)
for _ in range(2):
    a.copy_from(a0)
    f2.pls_recursive(a, cfg)
f2.timer_start()
for _ in range(steps):
    a.copy_from(a0)
    r = f2.pls_recursive(a, cfg)
ms = f2.timer_stop() / steps
print(f"n={n} rank={r.rank} digest={a.digest()} {ms:.3f} ms/step")
