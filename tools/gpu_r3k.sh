mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py -x -q > gpurun_out/r3k.log 2>&1; echo "rc=$?" >> gpurun_out/r3k.log
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q -k "c5a or c3 or c4" > gpurun_out/r3k_full.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_full.log
for c in c3 c4 c5a c2; do timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3k_$c.json 2>&1; done
