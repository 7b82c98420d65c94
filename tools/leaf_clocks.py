"""Phase clocks of k_leaf_pivot (needs tools/libf2gpu_prof.so built with -DF2_LEAF_PROFILE)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

L = f2.load_library("tools/libf2gpu_prof.so")
L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
for m, n in [(65536, 64), (65536, 128), (4096, 64), (128, 64)]:
    a = f2.DeviceMatrix(m, n)
    a.randomize(0.5, 7)
    for rep in range(3):
        b = a.clone()
        r = f2.mmpf_pls(b)
    out = (C.c_longlong * 16)()
    L.f2_debug_clocks(out, 16)
    print(m, n, "rank", r.rank, "clocks", list(out))
