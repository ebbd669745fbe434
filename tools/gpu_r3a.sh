mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_rare_paths.py -x -q > gpurun_out/r3a_par.log 2>&1; echo rc=$? >> gpurun_out/r3a_par.log
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q -k "c5b or 1d" > gpurun_out/r3a_full.log 2>&1; echo rc=$? >> gpurun_out/r3a_full.log
timeout 300 python bench.py --config c5b --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r3a_c5b.json 2>&1
