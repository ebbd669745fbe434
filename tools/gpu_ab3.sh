# A/B of prebuilt libraries over several configs: tools/gpu_ab3.sh "c5a c5b c4" lib...
CFGS=$1; shift
mkdir -p gpurun_out
for cfg in $CFGS; do
for rep in 1 2; do
for L in "$@"; do
    DMS_LIB=$PWD/abx/$L timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-d1 --no-e2e > gpurun_out/ab3.json 2>/dev/null
    python - <<PY
import json
d=json.load(open("gpurun_out/ab3.json")); s=d["stages_ms_per_step"]
print("$cfg $L rep$rep", d["ms_per_step"], "grad", s["gradient"], "order", s["order"], "crit", s["critical"], "d0", s["d0"], "dtop", s["dtop"])
PY
done
done
done
