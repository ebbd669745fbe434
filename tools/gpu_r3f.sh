mkdir -p gpurun_out
for v in "X=0" "DMS_ORDER_CTAS=1" "DMS_ORDER_CTAS=3"; do
  env $v timeout 300 python bench.py --config c3 --steps 5 --no-cpu-baseline --no-e2e --no-d1 > "gpurun_out/r3f_c3_$(echo $v | tr ' =' '__').json" 2>&1
done
for cfg in c4 c2; do timeout 300 python bench.py --config $cfg --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3f_$cfg.json 2>&1; done
DMS_ORDER_SEQ=1 timeout 300 python bench.py --config c2 --steps 5 --no-cpu-baseline --no-e2e --no-d1 > gpurun_out/r3f_c2_seq.json 2>&1
