"""Summarise an ncu source-page SASS csv (`ncu -i X --page source --csv --print-source sass`):
top instructions by warp-stall samples with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
num = lambda v: int(v) if v.isdigit() else 0
print("samples", sum(num(r[iS]) for r in data), "inst", sum(num(r[iE]) for r in data))
tot = {}
for r in data:
    for i in reasons:
        tot[hdr[i]] = tot.get(hdr[i], 0) + num(r[i])
print("by reason:", sorted(((v, k) for k, v in tot.items()), reverse=True)[:8])
for i in sorted(range(len(data)), key=lambda i: -num(data[i][iS]))[:n]:
    r = data[i]
    rs = sorted(((num(r[j]), hdr[j][6:]) for j in reasons), reverse=True)[:2]
    print(r[iS].rjust(6), r[iE].rjust(9), r[0][-5:], r[1].strip()[:55].ljust(55), "<-", data[i - 1][1].strip()[:40], rs)
