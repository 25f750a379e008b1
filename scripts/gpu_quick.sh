#!/bin/bash
# quick gpurun call: the tests matching $K, then one bench config
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
PFC_PARITY_LOG=gpurun_out/parity_q.jsonl timeout 1200 python -m pytest tests -q -m gpu -k "${K:-pair or full_size or update_touches or graph}" > gpurun_out/pytest_q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log
for cfg in ${CFGS:-c4rank}; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-proxy > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "bench $cfg rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$cfg.json'));print(d['value'],d['ms_per_step'],{k:v['ms_per_step'] for k,v in d['sections'].items()})"
done
