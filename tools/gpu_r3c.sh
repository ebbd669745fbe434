mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r3c_par.log 2>&1; echo rc=$? >> gpurun_out/r3c_par.log
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q -k "c5b" > gpurun_out/r3c_full.log 2>&1; echo rc=$? >> gpurun_out/r3c_full.log
timeout 300 python bench.py --config c5b --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r3c_c5b.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_path" --csv python bench.py --config c5b --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r3c.csv 2>&1
