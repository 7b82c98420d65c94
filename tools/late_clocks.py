"""CTA 0's per-iteration cycles in a late panel (panel 56) of the 64K^2 run.  Needs
tools/libf2gpu_prof.so built with -DF2_PANEL_PROFILE -DF2_LEAF_CLOCKS."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

L = f2.load_library(sys.argv[1] if len(sys.argv) > 1 else "tools/libf2gpu_prof.so")
L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
a0 = f2.DeviceMatrix(65536, 65536)
a0.randomize(0.5, 3)
for rep in range(2):
    a = a0.clone()
    f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
out = (C.c_longlong * 96)()
L.f2_debug_clocks(out, 96)
v = list(out)[64:88]
print("iteration starts (cycles from the first):", [x - v[0] for x in v if x])
print("per iteration:", [v[i + 1] - v[i] for i in range(len(v) - 1) if v[i + 1] and v[i]])
d = list(out)[:8]
print(f"iteration 5 of panel 56 (cycles): window build {d[2]-d[1]}, leaf {d[3]-d[2]}, to the barrier {d[4]-d[3]}, "
      f"barrier {d[5]-d[4]}, control word of the next iteration {out[64+6]-d[5]}")
