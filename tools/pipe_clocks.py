"""Cycle counts of the pipelined panel kernel's CTA 0 phases (leaf 2 of panel 0)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

L = f2.load_library()
L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
a0 = f2.DeviceMatrix(65536, 65536)
a0.randomize(0.5, 3)
for rep in range(2):
    a = a0.clone()
    f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
out = (C.c_longlong * 32)()
L.f2_debug_clocks(out, 32)
v = list(out)
print(f"window build {v[22]} clk, pivot loop+uf/linv {v[20]} clk, whole fast leaf {v[21]} clk, "
      f"barrier CTA0 {v[23]} clk, barrier CTA1 {v[24]} clk  (1965 clk = 1 us)")
