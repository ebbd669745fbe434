set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
for cfg in c4 c3; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_$cfg.json 2> gpurun_out/r2b_bench_$cfg.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_pool -c 1 -o gpurun_out/r2b_grad_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2b_ncu.log 2>&1
