"""pls_recursive 64K^2 time for several panel widths (development aid)."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

a0 = f2.DeviceMatrix(65536, 65536)
a0.randomize(0.5, 3)
for W in [int(x) for x in sys.argv[1:]] or [512, 768, 1024]:
    f2.set_panel_bits(W)
    best = 1e9
    for rep in range(3):
        a = a0.clone()
        f2.timer_start()
        f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
        best = min(best, f2.timer_stop())
    print(f"W={W}: {best:.2f} ms", flush=True)
