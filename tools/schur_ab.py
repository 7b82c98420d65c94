"""A/B the table-apply kernel builds on one Schur-sized launch:
C(65536 x 64512) ^= A(65536 x 1024) * B(1024 x 64512), all device-resident (no extraction).
usage: python tools/schur_ab.py lib1.so [lib2.so ...]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

for lib in sys.argv[1:]:
    f2._lib = None
    f2.load_library(lib)
    a = f2.DeviceMatrix(65536, 65536)
    a.randomize(0.5, 3)
    # C = columns 1024.., A = columns 0..1023, B = rows 0..1023 of the same matrix,
    # disjoint windows (rows 1024.. for C and A) so the call is the Schur update shape
    wc = a.window(1024, 1024, 65536, 65536)
    wa = a.window(1024, 0, 65536, 1024)
    b = f2.DeviceMatrix(1024, 64512)
    b.randomize(0.5, 4)
    ts = []
    for rep in range(4):
        f2.timer_start()
        f2.addmul(a, a, b, wc=wc, wa=wa)
        ts.append(f2.timer_stop())
    ms = min(ts[1:])
    print(f"{lib}: Schur-sized addmul {ms:.3f} ms = {2.0 * 64512 * 1024 * 64512 / (ms * 1e-3) / 1e12:.0f} Tbit-op/s",
          flush=True)
    del a, b
