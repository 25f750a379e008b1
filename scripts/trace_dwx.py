"""Summarise a k_dwx_t per-tile epilogue trace: median phase lengths (us). The trace needs the diagnostic build
(PFC_BUILD_TAG=diag PFC_NVCC_EXTRA=-DPFC_DWX_DIAG=1) run with PFC_LIB=.../libpfc-diag.so PFC_DWX_TRACE=1 PFC_DWX_TRACE_FILE=..."""
import csv
import statistics as st
import sys

rows = list(csv.DictReader(open(sys.argv[1] if len(sys.argv) > 1 else "dwx_trace.csv")))
cols = ["start", "d1_full", "cnt_ok", "staged", "wb_empty", "batch0", "update_done"]
t0 = min(int(r["start"]) for r in rows)
t1 = max(int(r["update_done"]) for r in rows if int(r["update_done"]))
print(f"tiles {len(rows)}  kernel span (first tile start -> last update) {(t1 - t0) / 1e3:.1f} us")
for a, b in zip(cols, cols[1:]):
    v = [(int(r[b]) - int(r[a])) / 1e3 for r in rows if int(r[b]) and int(r[a])]
    print(f"{a:>10} -> {b:<12} median {st.median(v):6.2f}  p90 {sorted(v)[int(0.9 * len(v))]:6.2f}")
per = {}
for r in rows:
    per.setdefault(r["cta"], []).append(r)
gaps = []
for c, rs in per.items():
    rs.sort(key=lambda r: int(r["tile"]))
    for a, b in zip(rs, rs[1:]):
        gaps.append((int(b["start"]) - int(a["start"])) / 1e3)
print(f"tile period median {st.median(gaps):.2f} us")
dp = [(int(r["dot_published"]) - int(r["start"])) / 1e3 for r in rows if int(r["dot_published"])]
if dp:
    print(f"dot partial published, from tile start: median {st.median(dp):.2f}")
