"""Summaries of an ncu report: key metrics + the hottest SASS lines by stall samples.
usage: python tools/ncu_view.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(*args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if not l.startswith("==") and not l.startswith("\"Kernel Name\"")]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


keys = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
        "Waves Per SM", "Grid Size", "Block Size", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"]
for r in run("--page", "details", "--csv"):
    if r.get("Metric Name") in keys:
        print(f'{r["Section Name"][:28]:28s} {r["Metric Name"]:36s} {r["Metric Value"]:>14s} {r["Metric Unit"]}')
src = run("--page", "source", "--csv")
if src:
    col = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[col] or 0) for r in src) or 1
    print(f"\n# total stall samples {tot:.0f}; top lines")
    for r in sorted(src, key=lambda r: -float(r[col] or 0))[:top]:
        s = float(r[col] or 0)
        print(f'{s/tot*100:5.1f}%  {r["Address"][-5:]}  {r["Source"].strip()[:90]}')
