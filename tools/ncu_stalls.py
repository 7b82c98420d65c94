"""Top SASS lines of an ncu report with their dominant stall reasons.
usage: python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
body = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in body) or 1
agg = {s: sum(float(r[s] or 0) for r in body) for s in stalls}
print("stall totals:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for r in sorted(body, key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    s = float(r["Warp Stall Sampling (All Samples)"] or 0)
    reasons = sorted(((float(r[k] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{s / tot * 100:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:58]:58s} " +
          " ".join(f"{n}:{v / max(s, 1) * 100:.0f}%" for v, n in reasons if v))
