"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def summary(path, out=sys.stdout):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, []])
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("f2g::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = {"nsecond": v / 1000, "ns": v / 1000, "usecond": v, "us": v, "msecond": v * 1000, "ms": v * 1000}[unit]
        a = agg[name]
        a[0] += 1
        a[1] += us
        a[2].append(us)
    tot = sum(a[1] for a in agg.values())
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        s = sorted(a[2])
        print(f"{k:28s} n={a[0]:5d} total={a[1]/1000:9.3f} ms share={a[1]/tot*100:5.1f}% "
              f"med={s[len(s)//2]:8.1f}us max={s[-1]:9.1f}us", file=out)
    print(f"total {tot/1000:.3f} ms over {len(rows)} launches", file=out)


if __name__ == "__main__":
    summary(sys.argv[1])
