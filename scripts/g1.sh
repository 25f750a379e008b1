mkdir -p gpurun_out/g1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1/tests.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/g1/bench_eform.json 2> gpurun_out/g1/bench_eform.err
PFC_EFORM=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/g1/bench_noef.json 2> gpurun_out/g1/bench_noef.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1
