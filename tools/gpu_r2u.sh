mkdir -p gpurun_out
python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/r2u_plain.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:"k_hist|k_scatter|k_win|k_scan_excl" --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/r2u_order.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scatter" -s 1 -c 1 -o gpurun_out/r2u_scatter python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/r2u_ncu2.log 2>&1
