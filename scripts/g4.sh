mkdir -p gpurun_out/g4
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pair_kernels or path_flags" > gpurun_out/g4/tests_pair.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g4/tests.log 2>&1
for i in 1 2; do
for ef in 1 0; do
PFC_EFORM=$ef timeout 300 python bench.py --config c4rank --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4rank ef$ef', d['ms_per_step'], ' '.join('%s=%.3f' % (k['kernel'], k['avg_ms']) for k in d['kernels']), d.get('sections'))" >> gpurun_out/g4/ab.log 2>&1
done; done
