set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py -x -q > gpurun_out/r2l_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_parity.log
for cfg in c4 c3; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2l_$cfg.json 2>&1
  DMS_ORDER_SEQ=1 timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2l_${cfg}_seq.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_gradient_pool -c 1 --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2l_ncu_grad.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none -k regex:k_gradient_pool -c 1 --csv python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2l_ncu_grad_c3.csv 2>&1
