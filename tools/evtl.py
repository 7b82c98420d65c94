"""Per-panel event timeline of one 64K^2 pls_recursive (non-graph run, F2_EVTL=1):
durations between consecutive marks on the main stream and the side-stream panel kernel.
usage: F2_NO_GRAPH=1 F2_EVTL=1 python tools/evtl.py [n]"""
import collections
import os
import subprocess
import sys

if os.environ.get("F2_EVTL") is None:
    env = dict(os.environ, F2_NO_GRAPH="1", F2_EVTL="1")
    out = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    lines = [l.split() for l in out.stderr.splitlines() if l.startswith("EVTL")]
    print(out.stdout.strip(), "rc", out.returncode)
    print("\n".join(l for l in out.stderr.splitlines() if not l.startswith("EVTL"))[-2000:])
    # keep the last run only (marks restart at "start")
    starts = [i for i, l in enumerate(lines) if l[2] == "start"]
    lines = lines[starts[-1]:]
    per = collections.defaultdict(dict)
    for _, p, name, t in lines:
        per[int(p)][name] = float(t)
    order = ["gather0", "gather1", "snapshot", "trsm_narrow", "schur_narrow", "trsm_wide", "schur_wide"]
    tot = collections.Counter()
    prev_end = per[-1].get("panel0", 0.0)
    rows = []
    for p in sorted(k for k in per if k >= 0):
        d = per[p]
        seg = {}
        last = prev_end
        for nm in order:
            if nm in d:
                seg[nm] = d[nm] - last
                last = d[nm]
        pk = d.get("panel_next", float("nan")) - d.get("schur_narrow", float("nan"))
        seg["panel_next(side)"] = pk
        end = max(d.get("schur_wide", last), d.get("panel_next", last), last)
        seg["join_wait"] = end - last
        prev_end = end
        for k, v in seg.items():
            if v == v:
                tot[k] += v
        rows.append((p, seg))
    for p, seg in rows:
        if p % 4 == 0 or p >= 60 or os.environ.get("EVTL_ALL"):
            print(f"panel {p:2d}: " + " ".join(f"{k}={v:7.1f}" for k, v in seg.items()))
    print("totals (us): " + " ".join(f"{k}={v:.0f}" for k, v in tot.items()))
    print(f"span {prev_end:.0f} us")
    sys.exit(0)

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
a0 = f2.DeviceMatrix(n, n)
a0.randomize(0.5, 3)
for rep in range(2):
    a = a0.clone()
    r = f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20))
print("rank", r.rank)
