"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel device time of the last search (the final `n` launches)."""
import csv
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = list(csv.reader(open(path)))
h = None
out = []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        out.append((d["Kernel Name"], float(d["Metric Value"])))
tot = 0.0
for name, v in out[-n:]:
    tot += v
    print(f"{v / 1000:8.1f} us  {name[:90]}")
print(f"{tot / 1000:8.1f} us  total of the last {n}")
