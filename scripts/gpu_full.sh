#!/bin/bash
# driver-like round: full GPU suite, default bench line, reference arm
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
PFC_PARITY_LOG=gpurun_out/parity_full.jsonl timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_full.log | tail -8
fi
T0=$SECONDS; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$? wall=$((SECONDS - T0)) s"
T0=$SECONDS; timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref_full.json 2> gpurun_out/ref_full.err
echo "ref rc=$? wall=$((SECONDS - T0)) s"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_full.json"))
print({k: d[k] for k in ("value", "ms_per_step", "gemm_tensor_frac")}, d["roofline"]["frac"], d["e2e"]["value"])
print("proxy", d["per_rank_proxy"]["ms_per_step"], d["per_rank_proxy"]["gemm_tensor_frac"])
r = json.load(open("gpurun_out/ref_full.json"))
print("ref", r["value"], r["ms_per_step"], r["steps"])
PY
