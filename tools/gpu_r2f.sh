set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2f_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_parity.log
for cfg in c4 c5b c5a c3; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f_$cfg.json 2>&1
  DMS_ORDER_SEQ=1 timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f_${cfg}_seq.json 2>&1
done
DMS_ORDER_SEQ=1 DMS_ORDER_CTAS=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_hist|k_scatter|k_scan|k_win" -c 16 --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2f_ncu_lsd.csv 2>&1
