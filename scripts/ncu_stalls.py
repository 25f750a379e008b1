"""Top SASS lines by warp-stall samples for one kernel (by launch index in the report) of an ncu report.
    python scripts/ncu_stalls.py report.ncu-rep <launch-index> [n]"""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", pat,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
h = rows[hi]; ci = {k: i for i, k in enumerate(h)}
key = [k for k in h if k.startswith("Warp Stall Sampling (All")][0]
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    try:
        v = float(r[ci[key]] or 0)
    except ValueError:
        continue
    data.append((v, r))
tot = sum(v for v, _ in data) or 1
tots = {s: sum(float(r[ci[s]] or 0) for _, r in data) for s in stalls}
print("stall totals:", {k[6:]: round(v / tot, 3) for k, v in sorted(tots.items(), key=lambda kv: -kv[1])[:8]})
data.sort(key=lambda t: -t[0])
for v, r in data[:n]:
    top = max(stalls, key=lambda s: float(r[ci[s]] or 0))
    print(f"{100*v/tot:5.1f}% {top[6:]:14s} {r[ci['Source']].strip()[:90]}")
