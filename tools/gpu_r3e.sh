mkdir -p gpurun_out
for v in "DMS_ORDER_SEQ=1" "DMS_ORDER_SEQ=0" "DMS_ORDER_SEQ=0 DMS_ORDER_CTAS=1" "DMS_ORDER_SEQ=0 DMS_ORDER_CTAS=3" "DMS_ORDER_SEQ=0 DMS_ORDER_CTAS=0"; do
  env $v timeout 300 python bench.py --config c4 --steps 5 --no-cpu-baseline --no-e2e --no-d1 > "gpurun_out/r3e_$(echo $v | tr ' =' '__').json" 2>&1
done
