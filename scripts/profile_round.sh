set -x
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/prof/tests.log
timeout 600 python bench.py > gpurun_out/prof/bench_c4.json 2> gpurun_out/prof/bench_c4.err
timeout 300 python bench.py --config c4rank --steps 30 --warmup 5 > gpurun_out/prof/bench_c4rank.json 2>/dev/null
timeout 300 python bench.py --config c4rank2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_c4rank2.json 2>/dev/null
timeout 300 python bench.py --config c4rank4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_c4rank4.json 2>/dev/null
timeout 300 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_c3.json 2>/dev/null
timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_c2.json 2>/dev/null
timeout 600 python bench.py --config c3 --params host --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c3_host.json 2>/dev/null
timeout 600 python bench.py --config c5rank --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c5rank.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:^k_ -c 300 --csv --log-file gpurun_out/prof/launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:^k_ -c 300 --csv --log-file gpurun_out/prof/launches_c4rank.csv python bench.py --config c4rank --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dwx_t|k_logits_gather" -s 2 -c 2 -o gpurun_out/prof/fused_c4 python scripts/prof_step.py 10000000 256 0.1 4 1 bf16 > gpurun_out/prof/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dw_sgd_pair|k_logits_pair" -s 2 -c 2 -o gpurun_out/prof/pair_c4rank python scripts/prof_step.py 1250000 2048 0.1 4 1 bf16 > gpurun_out/prof/ncu_full2.log 2>&1
ls -la gpurun_out/prof
