mkdir -p gpurun_out/g2
PFC_LIB=variants/local2/libpfc.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or eform or train" > gpurun_out/g2/tests_local2.log 2>&1
bash scripts/ab_run.sh c4 3 xch local1 local2 local4 > gpurun_out/g2/ab.log 2>&1
