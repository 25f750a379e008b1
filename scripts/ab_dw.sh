#!/bin/bash
# A/B of env-selected kernel variants at the per-rank C4 shape (and C4) with the same build; a variant is a
# '+'-separated list of NAME=VALUE settings
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in ${VARIANTS:-"PFC_DW_ORDER=0" "PFC_DW_ORDER=1"}; do
  for cfg in ${CFGS:-c4rank}; do
    env ${v//+/ } timeout 300 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-proxy > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v $cfg', d['ms_per_step'],{k:v['ms_per_step'] for k,v in d['sections'].items() if v['ms_per_step']>0.05})" || tail -3 gpurun_out/ab.err
  done
done
