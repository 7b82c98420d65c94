"""Kernel-family times (stats run) of one decomposition: python tools/fam.py m n kind [recursive|mmpf]"""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

m, n, kind = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
path = sys.argv[4] if len(sys.argv) > 4 else "recursive"
a0 = f2.DeviceMatrix(m, n)
if kind == "sparse":
    a0.fixed_weight(64, 5)
elif kind == "xy":
    x = f2.DeviceMatrix(m, m // 2)
    x.randomize(0.5, 4)
    y = f2.DeviceMatrix(m // 2, n)
    y.randomize(0.5, 5)
    a0 = f2.mul_m4rm(x, y)
else:
    a0.randomize(0.5, 1)
a = f2.DeviceMatrix(m, n)
run = (lambda: f2.mmpf_pls(a)) if path == "mmpf" else (lambda: f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20)))
for i in range(3):
    a.copy_from(a0)
    f2.timer_start()
    r = run()
    t = f2.timer_stop()
f2.stats_reset()
f2.stats_enable(True)
a.copy_from(a0)
run()
f2.stats_enable(False)
fam = {k: f2.stats_get(i) for i, k in enumerate(["schur", "panel", "trsm", "other"])}
print(f"{m}x{n} {kind} {path}: {t:.2f} ms, rank {r.rank}; stats: " +
      ", ".join(f"{k} {v['ms']:.2f} ms/{v['launches']}" for k, v in fam.items()))
