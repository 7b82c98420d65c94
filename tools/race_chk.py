"""Config-3 repeats with a debug build that self-checks the slot sources (-DF2_CHECK_SRC):
prints st->dbg[0..7] (mismatch count, panel word, leaf, slot, expected, got, kb) per bad run."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 20
L = f2.load_library()
L.f2_debug_clocks.argtypes = [C.POINTER(C.c_longlong), C.c_int]
want = int(json.load(open("tests/golden/configs.json"))["c3_dense_65536"]["recursive"]["packed_digest"])
cfg = f2.EliminationConfig(cutoff_bytes=2 << 20)
a0 = f2.DeviceMatrix(65536, 65536)
a0.randomize(0.5, 3)
a = f2.DeviceMatrix(65536, 65536)
for i in range(runs):
    a.copy_from(a0)
    r = f2.pls_recursive(a, cfg)
    d = a.digest()
    cl = (C.c_longlong * 32)()
    L.f2_debug_clocks(cl, 32)
    print(i, "ok" if d == want else "BAD", r.rank, list(cl)[:8], flush=True)
