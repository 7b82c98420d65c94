"""A 65536 x 2048 pls_recursive (two panels) for profiling the panel kernel (k_panel_pipe)."""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

a0 = f2.DeviceMatrix(65536, 2048)
a0.randomize(0.5, 7)
for _ in range(2):
    a = a0.clone()
    r = f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=1 << 10))
print("rank", r.rank)
