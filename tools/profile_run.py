"""One PLS call for profiling: python tools/profile_run.py N [recursive|mmpf] [warm]"""
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
entry = sys.argv[2] if len(sys.argv) > 2 else "recursive"
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
a0 = f2.DeviceMatrix(n, n)
a0.randomize(0.5, 3)
for _ in range(warm + 1):
    a = a0.clone()
    r = f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20)) if entry == "recursive" else f2.mmpf_pls(a)
print("rank", r.rank, "launches", f2.last_launch_count())
