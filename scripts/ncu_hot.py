"""Top stalled SASS instructions of an ncu report's source page (ncu -i X --page source --csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci, si = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((float(r[ci]), i, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for v, i, s in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  #{i:5d}  {s[:100]}")
