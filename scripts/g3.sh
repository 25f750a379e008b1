mkdir -p gpurun_out/g3
for v in xch local2; do
 for ef in 1 0; do
  PFC_LIB=variants/$v/libpfc.so PFC_EFORM=$ef timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_dwx|k_logits_gather|k_softmax|k_eform" -c 40 --csv --log-file gpurun_out/g3/launch_${v}_ef$ef.csv python scripts/prof_step.py 10000000 256 0.1 8 1 bf16 > /dev/null 2>&1
 done
done
PFC_EFORM=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dwx_t" -s 2 -c 1 -o gpurun_out/g3/dwx_ef1 python scripts/prof_step.py 10000000 256 0.1 4 1 bf16 > gpurun_out/g3/n1.log 2>&1
PFC_EFORM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dwx_t" -s 2 -c 1 -o gpurun_out/g3/dwx_ef0 python scripts/prof_step.py 10000000 256 0.1 4 1 bf16 > gpurun_out/g3/n0.log 2>&1
