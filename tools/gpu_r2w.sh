mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py -x -q > gpurun_out/r2w_par.log 2>&1; echo rc=$? >> gpurun_out/r2w_par.log
for cfg in c4 c3 c5a c5b; do
  timeout 300 python bench.py --config $cfg --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r2w_$cfg.json 2>&1
  DMS_ORDER_OS=0 timeout 300 python bench.py --config $cfg --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r2w_${cfg}_old.json 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_os" --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/r2w_os.csv 2>&1
