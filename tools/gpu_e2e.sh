# e2e A/B of the host-input path's order grid (c4, c3)
mkdir -p gpurun_out
for cfg in c4 c3; do
for e in DMS_HOST_ORDER_BESIDE=1 DMS_HOST_ORDER_BESIDE=0 "DMS_HOST_ORDER_BESIDE=1 DMS_ORDER_CTAS=2"; do
  env $e timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-d1 > gpurun_out/e2e_ab.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/e2e_ab.json"))
print("$cfg $e", "dev", d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], d["e2e"]["value"])
PY
done
done
