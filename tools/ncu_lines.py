"""Per CUDA source line stall samples / executed instructions from an ncu report
(needs -lineinfo).  usage: python tools/ncu_lines.py report.ncu-rep [top] [file-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path = None
stats = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and r[0] != "":  # a CUDA source line row
        try:
            stats.append((path, int(r[0]), r[1], float(r[4] or 0), float(r[7] or 0)))
        except (ValueError, IndexError):
            pass
tot = sum(s[3] for s in stats) or 1
for p, ln, src, samp, inst in sorted(stats, key=lambda s: -s[3])[:top]:
    if filt and filt not in p:
        continue
    print(f"{samp / tot * 100:5.1f}% inst={inst:10.0f} {p.split('/')[-1]}:{ln:<4d} {src.strip()[:90]}")
