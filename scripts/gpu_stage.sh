#!/bin/bash
# staged gpurun call: short sanity of the new paths first (kill early on a hang), then the given pytest selection
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 240 python scripts/sanity_new.py > gpurun_out/sanity.log 2>&1
rc=$?
echo "sanity rc=$rc"; tail -12 gpurun_out/sanity.log
[ $rc -ne 0 ] && exit $rc
if [ -n "$PROBE" ]; then timeout 120 python scripts/gather_probe.py > gpurun_out/probe.log 2>&1; cat gpurun_out/probe.log; fi
PFC_PARITY_LOG=gpurun_out/parity_s.jsonl timeout ${PT_TIMEOUT:-900} python -m pytest ${TESTS:-tests} -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/pytest_s.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_s.log | tail -15
for cfg in ${CFGS:-}; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-proxy > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "bench $cfg rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$cfg.json'));print(d['value'],d['ms_per_step'],{k:v['ms_per_step'] for k,v in d['sections'].items()})"
done
