mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rare_paths.py tests/test_gpu_fullsize_oracle.py -x -q -k "not c4 and not c3" > gpurun_out/r3d.log 2>&1; echo rc=$? >> gpurun_out/r3d.log
timeout 300 python bench.py --config c5b --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r3d_c5b.json 2>&1
