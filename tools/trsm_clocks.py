"""Phase clocks of k_pivot_trsm (panel mode, CTA 0) from tools/libf2gpu_prof.so."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

L = f2.load_library("tools/libf2gpu_prof.so")
for n in (2048, 4096):
    a = f2.DeviceMatrix(n, n)
    a.randomize(0.5, 7)
    for rep in range(2):
        b = a.clone()
        r = f2.pls_recursive(b, f2.EliminationConfig(cutoff_bytes=2 << 20))
    out = (C.c_longlong * 32)()
    L.f2_debug_clocks(out, 32)
    print(n, "clocks", list(out)[16:])
