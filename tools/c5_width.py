"""Config 5's shape at several widths: how much the panels past full row rank cost.
python tools/c5_width.py"""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

m = 16384
for n in (16384, 32768, 65536, 131072):
    a0 = f2.DeviceMatrix(m, n)
    a0.fixed_weight(64, 5)
    best = 1e9
    for rep in range(4):
        a = a0.clone()
        f2.timer_start()
        r = f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
        best = min(best, f2.timer_stop())
    print(f"{m}x{n}: rank {r.rank}, {best:.2f} ms, launches {f2.last_launch_count()}", flush=True)
