#!/bin/bash
# ncu of the dW + SGD kernels at the per-rank C4 shape: the pair kernel (default) and the all-column kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --config c4rank --steps 3 --warmup 3 --no-cpu-baseline --no-proxy"
$CMD > gpurun_out/plain_pair.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dw_sgd_pair -s 2 -c 1 -o gpurun_out/prof_dwpair $CMD > gpurun_out/ncu_pair.log 2>&1
echo "pair rc=$?"
PFC_DWFULL=1 $CMD > gpurun_out/plain_full.log 2>&1 && \
PFC_DWFULL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dw_sgd_full -s 2 -c 1 -o gpurun_out/prof_dwfull $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
