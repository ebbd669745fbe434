mkdir -p gpurun_out
python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/r2v_plain.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gradient_pool" -c 1 -o gpurun_out/r2v_grad python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/r2v_ncu.log 2>&1
