"""Per-panel timeline (us from the first panel kernel start): panel kernel [start, end] and
the trailing Schur [start, end].  Needs tools/libf2gpu_tl.so built with -DF2_TIMELINE."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

L = f2.load_library("tools/libf2gpu_tl.so")
L.f2_debug_timeline.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
a0 = f2.DeviceMatrix(65536, 65536)
a0.randomize(0.5, 3)
for rep in range(2):
    a = a0.clone()
    f2.timer_start()
    f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
    ms = f2.timer_stop()
out = (C.c_ulonglong * 512)()
L.f2_debug_timeline(out, 512)
v = [list(out[i * 128:(i + 1) * 128]) for i in range(4)]
t0 = v[0][0]
print(f"total {ms:.2f} ms")
for p in [0, 1, 40, 41, 56, 57, 58, 59, 60, 61, 62, 63]:
    ps, pe, ss, se = v[0][p], v[1][p], v[2][p], v[3][p]
    f = lambda x: (x - t0) / 1000 if 0 < x < (1 << 63) else float('nan')
    print(f"panel {p:2d}: kernel {f(ps):9.1f} .. {f(pe):9.1f} ({(pe - ps) / 1000:6.1f})   schur {f(ss):9.1f} .. {f(se):9.1f}")
