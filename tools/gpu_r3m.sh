mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_rare_paths.py -x -q > gpurun_out/r3m.log 2>&1; echo "rc=$?" >> gpurun_out/r3m.log
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q -k "c5b or c5a or c3" > gpurun_out/r3m_full.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_full.log
for c in c4 c3 c5a c5b c2; do timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3m_$c.json 2>&1; done
