set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_pool -c 1 -o gpurun_out/r2i_grad_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2i_ncu.log 2>&1
