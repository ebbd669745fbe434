set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
for cfg in c4 c3; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_$cfg.json 2> gpurun_out/r2a_bench_$cfg.err
  DMS_GRAD_FAST=0 timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a_bench_${cfg}_old.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gradient_pool -c 1 --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2a_ncu_grad.csv 2>&1
