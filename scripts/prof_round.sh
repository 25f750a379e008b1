#!/bin/bash
# round-2 profiles: per-launch device times + DRAM bytes of the bench step (C4 on one GPU, and the per-rank C4 shape),
# then one full capture each of the top kernels (k_dwx_t at C4, k_logits_gather at C4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for cfg in c4 c4rank; do
  CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-proxy"
  $CMD > gpurun_out/plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv $CMD > gpurun_out/ncu_$cfg.log 2>&1
  echo "$cfg launches rc=$?"
done
CMD="python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-proxy"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dwx_t|k_logits_gather" -s 20 -c 2 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full_c4.log 2>&1
echo "c4 full rc=$?"
