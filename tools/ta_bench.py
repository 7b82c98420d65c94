"""HBM rate of the MMPF table-apply (f2_addmul with K <= 64) over a 1 GiB C: C 65536 x 131072."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

rows, cols = 65536, 131072
c = f2.DeviceMatrix(rows, cols)
c.randomize(0.5, 11)
for kbits in [int(x) for x in sys.argv[1:]] or [8, 64]:
    am = f2.DeviceMatrix(rows, kbits)
    am.randomize(0.5, 12)
    bm = f2.DeviceMatrix(kbits, cols)
    bm.randomize(0.5, 13)
    for _ in range(3):
        f2.addmul(c, am, bm)
    f2.stats_reset()
    f2.stats_enable(True)
    for _ in range(5):
        f2.addmul(c, am, bm)
    f2.stats_enable(False)
    st = f2.stats_get(0)
    print(f"K={kbits}: {st['ms'] / st['launches']:.3f} ms, {st['bytes'] / (st['ms'] / 1e3) / 1e9:.0f} GB/s")
