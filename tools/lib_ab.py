"""A/B of library builds: config 3 and config 2 device times (best of reps).  python tools/lib_ab.py lib1.so lib2.so ..."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

for rnd in range(2):
    for lib in sys.argv[1:]:
        f2._lib = None
        f2.load_library(lib)
        out = []
        for n in (65536, 16384):
            a0 = f2.DeviceMatrix(n, n)
            a0.randomize(0.5, 3)
            ts = []
            for rep in range(6):
                a = a0.clone()
                f2.timer_start()
                f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
                ts.append(f2.timer_stop())
            out.append(f"n={n}: min {min(ts[1:]):.3f} med {sorted(ts[1:])[2]:.3f} ms")
            del a0, a
        print(lib, "; ".join(out), flush=True)
