#!/bin/bash
# host-resident (f4) and fused-collective (f2, world 1) bench lines, then full ncu captures at the per-rank C4 shape
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # name, args...
  local n=$1; shift
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-proxy "$@" > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err
  python -c "import json;d=json.load(open('gpurun_out/b_$n.json'));print('$n', d['value'], d['ms_per_step'], {k:v['ms_per_step'] for k,v in d['sections'].items() if v['ms_per_step']>0.02})" || tail -3 gpurun_out/b_$n.err
}
run c3_dev --config c3
run c3_host --config c3 --params host
PFC_HOST_STAGE=0 run c3_host_zc --config c3 --params host
run c4rank_host --config c4rank --params host
PFC_HOST_STAGE=0 run c4rank_host_zc --config c4rank --params host
run c4rank_fused --config c4rank --comm nccl_fused
run c2_fused --config c2 --comm nccl_fused
run c2 --config c2
CMD="python bench.py --config c4rank --steps 3 --warmup 3 --no-cpu-baseline --no-proxy"
$CMD > gpurun_out/plain_c4rank.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dw_sgd_pairx|k_logits_pair|k_tc_gemm" -s 12 -c 3 -o gpurun_out/prof_c4rank $CMD > gpurun_out/ncu_full_c4rank.log 2>&1
echo "c4rank full rc=$?"
