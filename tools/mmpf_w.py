"""mmpf_pls device time by panel width (F2_MMPF_PANEL_BITS): python tools/mmpf_w.py m n [kind]"""
import os
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

m, n = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "dense"
a0 = f2.DeviceMatrix(m, n)
if kind == "sparse":
    a0.fixed_weight(64, 5)
else:
    a0.randomize(0.5, 1)
a = f2.DeviceMatrix(m, n)
ts = []
for i in range(6):
    a.copy_from(a0)
    f2.timer_start()
    r = f2.mmpf_pls(a)
    ts.append(f2.timer_stop())
print(f"W={os.environ.get('F2_MMPF_PANEL_BITS', '64')} {m}x{n} {kind} rank {r.rank} digest {a.digest()} "
      f"{sorted(ts)[len(ts) // 2]:.2f} ms")
