"""Cost of a graph-cache miss: six matrix buffers factored in turn (four cache slots), 16K^2 and 64K^2."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

for n, nb in ((16384, 6), (65536, 6)):
    a0 = f2.DeviceMatrix(n, n)
    a0.randomize(0.5, 3)
    want = None
    bufs = [f2.DeviceMatrix(n, n) for _ in range(nb)]
    for rnd in range(3):
        ts = []
        for b in bufs:
            b.copy_from(a0)
            f2.timer_start()
            r = f2.pls_recursive(b, f2.EliminationConfig(cutoff_bytes=2 << 20))
            ts.append(f2.timer_stop())
            d = (r.rank, b.digest())
            want = want or d
            assert d == want
        print(n, "round", rnd, " ".join(f"{t:.1f}" for t in ts), flush=True)
    del bufs, a0
