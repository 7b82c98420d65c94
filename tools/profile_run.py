"""One PLS call for profiling: python tools/profile_run.py N [recursive|mmpf] [warm] [sparse M]
(sparse: config 5's shape, M x N with 64 ones per row, seed 5)"""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
entry = sys.argv[2] if len(sys.argv) > 2 else "recursive"
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if len(sys.argv) > 4 and sys.argv[4] == "sparse":
    m = int(sys.argv[5])
    a0 = f2.DeviceMatrix(m, n)
    a0.fixed_weight(64, 5)
else:
    a0 = f2.DeviceMatrix(n, n)
    a0.randomize(0.5, 3)
for _ in range(warm + 1):
    a = a0.clone()
    r = f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20)) if entry == "recursive" else f2.mmpf_pls(a)
print("rank", r.rank, "launches", f2.last_launch_count())
