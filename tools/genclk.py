"""Clock accounting of the panel kernel's general search on config 5's first panel
(tools/libf2gpu_prof.so built with -DF2_LEAF_CLOCKS): dbg[0] window-loop cycles, [1] scan
cycles, [3] scans, [5] scans from the compact list, [4] list size (last leaf), [6] total
cycles in the general search, [7] general leaves -- summed over panel 0's leaves."""
import ctypes as C, sys
sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2
L = f2.load_library(sys.argv[1] if len(sys.argv) > 1 else "tools/libf2gpu_prof.so")
L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
a = f2.DeviceMatrix(16384, 131072); a.fixed_weight(64, 5)
b = a.clone()
f2.pls_recursive(b, f2.EliminationConfig(cutoff_bytes=2 << 20))
cl = (C.c_longlong * 32)(); L.f2_debug_clocks(cl, 32)
print({k: cl[k] for k in range(16)})
