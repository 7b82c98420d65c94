"""globaltimer stamps of k_panel_leaves (first panel, leaf 1) and the K1 internals.
Needs tools/libf2gpu_prof.so built with -DF2_PANEL_PROFILE -DF2_LEAF_CLOCKS:
  nvcc <NVCC_FLAGS of __graft_entry__> -DF2_PANEL_PROFILE -DF2_LEAF_CLOCKS -o tools/libf2gpu_prof.so paper_1006_1744_b200/csrc/*.cu"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

L = f2.load_library("tools/libf2gpu_prof.so")
L.f2_debug_prof.argtypes = [C.POINTER(C.c_longlong), C.c_int]
names = {0: "iteration start", 1: "window built", 2: "fast leaf done", 3: "ctl written", 16: "transposed",
         18: "pivot loop + uf/linv", 19: "src/basis", 21: "tables/t16", 22: "lmap/U/P", 17: "loop done"}
names_old = {0: "leaf start", 10: "k1 window loaded", 11: "k1 outputs start", 12: "k1 st written", 1: "pivot done",
         2: "solve done", 3: "barrier 1 passed", 4: "update prep done", 5: "update done (CTA 0)",
         50: "tile rows loaded", 51: "tile finalized", 52: "tile lookups done"}
names.update({40 + g: f"solve group {g}" for g in range(8)})
names.update({15: "fast window loaded", 16: "fast transposed", 17: "fast loop done", 18: "fast rows out",
              19: "fast outputs done"})
names.update({15: "fast phys loaded", 16: "fast transposed", 17: "fast loop done", 18: "fast replay joined",
              19: "fast src done", 20: "fast outputs done", 21: "fast pivot rows written",
              22: "fast U computed (t0)", 23: "fast U sync"})
for m, n in [(65536, 2048)]:
    a = f2.DeviceMatrix(m, n)
    a.randomize(0.5, 7)
    for rep in range(3):
        b = a.clone()
        f2.pls_recursive(b, f2.EliminationConfig(cutoff_bytes=1 << 10))
    out = (C.c_longlong * 64)()
    L.f2_debug_prof(out, 64)
    v = list(out)
    print(m, n)
    L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
    cl = (C.c_longlong * 32)()
    L.f2_debug_clocks(cl, 32)
    for k in sorted((k for k in names if v[k]), key=lambda k: v[k]):
        print(f"  {names[k]:22s} {(v[k] - v[0]) / 1000:8.2f} us   clk {cl[k & 31] - cl[0]}")
