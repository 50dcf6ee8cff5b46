"""Stall samples per CUDA source line from an ncu source export
(--page source --csv --print-source=cuda,sass): python tools/src_hot.py f.csv [file-substring] [n]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur_file, hdr = "", None
agg, text, tot = defaultdict(float), {}, 0.0
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    tot += v
    if want in cur_file and r[0]:
        key = (cur_file.split("/")[-1], int(r[0]))
        agg[key] += v
        text[key] = r[1]
print(f"total samples {tot:.0f}")
for k in sorted(sorted(agg, key=lambda k: -agg[k])[:n]):
    print(f"{k[0]}:{k[1]:5d} {agg[k]:6.0f} {100 * agg[k] / tot:5.1f}%  {text[k].strip()[:90]}")
