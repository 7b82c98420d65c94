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
f = lambda x: (x - t0) / 1000 if 0 < x < (1 << 63) else float('nan')
print(f"total {ms:.2f} ms; engine span {f(max(v[1][:64])):.1f} us")
tot_t2 = tot_k = tot_gap = 0.0
for p in range(63):
    ks, ke = f(v[0][p + 1]), f(v[1][p + 1])
    ss, se = f(v[2][p]), f(v[3][p])
    nxt = f(v[2][p + 1]) if p + 1 < 62 else f(v[0][p + 2]) if p + 2 < 64 else float('nan')
    gap = (nxt - max(se, ke)) if nxt == nxt and se == se else float('nan')
    if p % 6 == 0 or p > 56:
        print(f"panel {p:2d}: schur t2 {ss:9.1f}..{se:9.1f} ({se - ss:6.1f})  kernel(p+1) {ks:9.1f}..{ke:9.1f} ({ke - ks:6.1f})  next-start gap {gap:6.1f}")
