set -x
mkdir -p gpurun_out
DMS_ORDER_SAMPLE=0 DMS_ORDER_SEQ=1 DMS_ORDER_CTAS=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_hist|k_scatter|k_scan" -c 12 --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2e_ncu_lsd.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ord_bucket|k_ord_count|k_ord_scatter" -c 3 -o gpurun_out/r2e_ord -f python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2e_ncu_ord.log 2>&1
