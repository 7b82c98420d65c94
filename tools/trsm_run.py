"""One 65536 x 65536 pls_recursive, for profiling the panel TRSM / gather kernels."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

a = f2.DeviceMatrix(65536, 65536)
a.randomize(0.5, 7)
r = f2.pls_recursive(a, f2.EliminationConfig())
print("rank", r.rank)
