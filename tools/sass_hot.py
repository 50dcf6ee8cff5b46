"""Top stalled SASS instructions of one kernel from an ncu --page source
--csv --print-source=sass export: python tools/sass_hot.py file.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(h) and r[ia] != "Address"]
body = [r for r in body if r[iss].replace(".", "").isdigit()]
tot = sum(float(r[iss] or 0) for r in body)
print(f"total samples {tot:.0f}")
order = sorted(range(len(body)), key=lambda i: -float(body[i][iss] or 0))[:n]
for i in sorted(order):
    r = body[i]
    print(f"{i:5d} {float(r[iss]):7.0f} {100*float(r[iss])/tot:5.1f}%  {r[isrc].strip()}")
