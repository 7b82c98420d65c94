"""e2e timing of the host-buffer entry point on config 3 (65536^2, seed 3) with the bench's
method (pinned buffers, f2 timer around the call), plus the packed digest check.
python tools/e2e.py [steps]   (tuning from the F2_* environment)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1006_1744_b200 as f2

N = 65536
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "configs.json")))
want = int(gold["c3_dense_65536"]["recursive"]["packed_digest"])
a = f2.DeviceMatrix(N, N)
a.randomize(0.5, 3)
words = N // 64
h0 = f2.pinned_empty((N, words))
a.download(h0)
del a
h = f2.pinned_empty((N, words))
cfg = f2.EliminationConfig(cutoff_bytes=2 << 20)
ts = []
for i in range(steps + 1):
    np.copyto(h, h0)
    f2.timer_start()
    f2.pls_recursive_host(h, N, cfg)
    ts.append(f2.timer_stop())
chk = f2.DeviceMatrix.from_host(h, N)
env = {k: v for k, v in os.environ.items() if k.startswith("F2_")}
print(json.dumps({"env": env, "ms": [round(t, 3) for t in ts[1:]], "median": round(float(np.median(ts[1:])), 3),
                  "digest_ok": chk.digest() == want}))
