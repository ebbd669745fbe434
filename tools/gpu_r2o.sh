set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2o_bench_c4.json 2> gpurun_out/r2o_bench_c4.err
for cfg in c3 c2; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2o_bench_$cfg.json 2> gpurun_out/r2o_bench_$cfg.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_d1 --log-file gpurun_out/r2o_d1_launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2o_ncu_l.log 2>&1
