#!/bin/bash
# A/B timing: alternate bench.py runs over the variant libraries given as arguments (variants/<name>/libpfc.so).
#   scripts/ab_run.sh <config> <reps> name1 name2 ...
cfg=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for v in "$@"; do
    PFC_LIB=variants/$v/libpfc.so timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], ' '.join('%s=%.3f' % (k['kernel'], k['avg_ms']) for k in d['kernels']))"
  done
done
