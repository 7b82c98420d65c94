"""A/B of library builds on the pipelined panel kernel: CTA 0 leaf-2 cycles and full 64K^2 time.
usage: python tools/pipe_ab.py lib1.so lib2.so ..."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

for lib in sys.argv[1:]:
    f2._lib = None
    L = f2.load_library(lib)
    L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
    a0 = f2.DeviceMatrix(65536, 65536)
    a0.randomize(0.5, 3)
    best = 1e9
    for rep in range(3):
        a = a0.clone()
        f2.timer_start()
        f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
        best = min(best, f2.timer_stop())
    out = (C.c_longlong * 32)()
    L.f2_debug_clocks(out, 32)
    v = list(out)
    print(f"{lib}: {best:.2f} ms; leaf2 (cumulative clk from the search start): window {v[22]} | loop+uf {v[20]} "
          f"| src/fb {v[25]} (linv {v[28]} src {v[29]} fb {v[30]}) | tables/t16 {v[26]} | lmap/U {v[27]} | leaf {v[21]}", flush=True)
    del a0, a
