mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rare_paths.py tests/test_gpu_parity.py -x -q > gpurun_out/r3h.log 2>&1; echo "rc=$?" >> gpurun_out/r3h.log
DMS_CHECK_INVARIANTS=1 timeout 300 python bench.py --config c4 --steps 2 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3h_inv_c4.json 2>&1
for c in c5b c3; do DMS_CHECK_INVARIANTS=1 timeout 300 python bench.py --config $c --steps 2 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3h_inv_$c.json 2>&1; done
timeout 300 python bench.py --config c4 --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3h_c4.json 2>&1
