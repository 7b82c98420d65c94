"""Phase clocks of the panel kernel (leaf 2 of the first panel).  Needs tools/libf2gpu_prof.so built with
-DF2_PANEL_PROFILE -DF2_LEAF_CLOCKS (nvcc <flags of __graft_entry__> ... -o tools/libf2gpu_prof.so csrc/*.cu)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2
L = f2.load_library(sys.argv[1] if len(sys.argv) > 1 else "tools/libf2gpu_prof.so")
L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
for m, n in [(65536, 2048), (16384, 2048)]:
    a = f2.DeviceMatrix(m, n); a.randomize(0.5, 7)
    for rep in range(3):
        b = a.clone(); f2.pls_recursive(b, f2.EliminationConfig(cutoff_bytes=1 << 10))
    cl = (C.c_longlong * 32)(); L.f2_debug_clocks(cl, 32)
    print(m, n, {k: cl[k] for k in list(range(8, 18)) + list(range(20, 32))})
