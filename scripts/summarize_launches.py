"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per launch) per kernel, and write
profiles/ncu_traffic.json for bench.py's `traffic` field.
    python scripts/summarize_launches.py launches.csv out_summary.csv [workload] [n_gpus]"""
import collections, csv, json, re, sys
src, out = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else "c4"
ngpu = int(sys.argv[4]) if len(sys.argv) > 4 else 1
rows = [r for r in csv.reader(open(src)) if r]
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ci = {n: i for i, n in enumerate(h)}
data = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    data[(r[ci['ID']], r[ci['Kernel Name']])][r[ci['Metric Name']]] = (float(r[ci['Metric Value']].replace(',', '')), r[ci['Metric Unit']])
mult = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-3, 'us': 1, 'ms': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, name), m in data.items():
    mt = re.search(r'(?:pfc::|unnamed>::)(?:<unnamed>::)?(k_[a-z0-9_]+(<[^>]*>)?)', name)
    if not mt:            # torch's own kernels (the synthetic W fill before the timed steps)
        continue
    short = mt.group(1)
    a = agg[short]; a[0] += 1
    t = m['gpu__time_duration.sum']; a[1] += t[0] * mult[t[1]]
    for mm, idx in (('dram__bytes_read.sum', 2), ('dram__bytes_write.sum', 3)):
        v, u = m[mm]; a[idx] += v * mult[u]
tot = sum(a[1] for a in agg.values())
sec = {'k_tc_gemm<5>': 'dw_gemm_sgd', 'k_tc_gemm<6>': 'dw_gemm_sgd', 'k_tc_gemm<0>': 'logits_gemm',
       'k_tc_gemm<1>': 'dx_gemm', 'k_gather_w<1>': 'gather_w', 'k_softmax_grad<1, 1>': 'softmax_grad',
       'k_logits_gather': 'gather_logits', 'k_dwx_t<1>': 'dwx_sgd', 'k_dwx_t<0>': 'dwx_sgd',
       'k_dw_sgd_pair<1>': 'dw_gemm_sgd', 'k_dw_sgd_pair<0>': 'dw_gemm_sgd', 'k_logits_pair': 'logits_gemm',
       # E-form train step (template <HINT, EF> / <EF>)
       'k_dwx_t<1, 1>': 'dwx_sgd', 'k_dwx_t<1, 0>': 'dwx_sgd', 'k_dwx_t<0, 1>': 'dwx_sgd', 'k_dwx_t<0, 0>': 'dwx_sgd',
       'k_logits_gather<1>': 'gather_logits', 'k_logits_gather<0>': 'gather_logits',
       'k_logits_pair<1>': 'logits_gemm', 'k_logits_pair<0>': 'logits_gemm', 'k_eform_dotw': 'eform_dotw',
       'k_logits_pair<1, 1>': 'logits_gemm', 'k_logits_pair<0, 1>': 'logits_gemm', 'k_logits_pair<1, 0>': 'logits_gemm',
       'k_logits_pair<0, 0>': 'logits_gemm', 'k_dw_sgd_pairx<1>': 'dw_gemm_sgd', 'k_dw_sgd_pairx<0>': 'dw_gemm_sgd',
       'k_dw_sgd_full<1>': 'dw_gemm_sgd', 'k_dw_sgd_full<0>': 'dw_gemm_sgd'}
lines = [f"# ncu launch list summary of {src} (workload {workload}, {ngpu} GPU): cold-cache, serialised launches",
         "# k_logits_gather = K5+K6 (gather, norms, fp16 operand, logits), k_dwx_t = K9+K11+K12 (dW, momentum SGD, dX) at M <= 256;",
         "# k_tc_gemm<0> = logits (K6), <1> = dx split-K (K9), <5>/<6> = dW + fused momentum SGD (K11+K12) otherwise",
         "kernel, launches, avg_us, share_of_step, dram_read_MB_per_launch, dram_write_MB_per_launch"]
traffic = {}
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{name}, {a[0]}, {a[1]/a[0]:.1f}, {a[1]/tot:.3f}, {a[2]/a[0]/1e6:.1f}, {a[3]/a[0]/1e6:.1f}")
    base = {'k_logits_gather': 'gather_logits', 'k_dwx_t': 'dwx_sgd', 'k_dwx_ring': 'dwx_sgd',
            'k_logits_pair': 'logits_gemm', 'k_dw_sgd_pairx': 'dw_gemm_sgd'}.get(name.split('<')[0])
    if name in sec or base:
        traffic[sec.get(name, base)] = round((a[2] + a[3]) / a[0])
open(out, 'w').write("\n".join(lines) + "\n")
tp = 'profiles/ncu_traffic.json'
try:
    tj = json.load(open(tp))
except (OSError, ValueError):
    tj = {}
wl = tj.get("workloads", {})
wl[f"{workload}/{ngpu}"] = {"workload": workload, "n_gpus": ngpu,
                            "source": src + " (ncu dram__bytes_read.sum + dram__bytes_write.sum per launch)",
                            "bytes_per_launch": traffic}
json.dump({"workloads": wl}, open(tp, 'w'), indent=1)
print("\n".join(lines[2:10]))
