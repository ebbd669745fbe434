mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_oracle.py -x -q -k "not c4" > gpurun_out/r2y_par.log 2>&1; echo rc=$? >> gpurun_out/r2y_par.log
for cfg in c4 c5b c5a c3; do
  timeout 300 python bench.py --config $cfg --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r2y_${cfg}_v1.json 2>&1
done
