#!/bin/bash
# launch lists (application replay: the 41 GB W/V shard is not saved/restored per kernel) of the bench step at C4
# and at the per-rank C4 shape, plus the per-rank C5 bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for cfg in ${PCFGS:-c4rank c4}; do
  CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-proxy"
  $CMD > gpurun_out/plain_$cfg.log 2>&1 && \
  timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_$cfg.csv $CMD > gpurun_out/ncu_$cfg.log 2>&1
  echo "$cfg launches rc=$?"
done
timeout 600 python bench.py --config c5rank --steps 10 --warmup 3 --no-cpu-baseline --no-proxy > gpurun_out/bench_c5rank.json 2>&1; echo "c5rank rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_c5rank.json'));print(d['ms_per_step'], d['value'], d['gemm_tensor_frac'])"
