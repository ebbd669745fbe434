set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q -k "midsize or c3" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
for o in 1 2 3 4 0; do
  DMS_ORDER_CTAS=$o timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_c4_octas$o.json 2>&1
done
DMS_ORDER_SEQ=1 timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_c4_seq.json 2>&1
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/r2c_c4_full.json 2>&1
