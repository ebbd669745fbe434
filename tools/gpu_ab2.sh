# A/B of env settings x prebuilt libraries on bench c4: tools/gpu_ab2.sh TAG "ENV1=..;ENV2=.." lib...
T=$1; shift
ENVS=$1; shift
mkdir -p gpurun_out
IFS=';' read -ra EV <<< "$ENVS"
for rep in 1 2; do
for L in "$@"; do
  for e in "${EV[@]}"; do
    env $e DMS_LIB=$PWD/abx/$L timeout 600 python bench.py --config ${CFG:-c4} --no-cpu-baseline --no-d1 --no-e2e > gpurun_out/ab_${T}.json 2>/dev/null
    python - <<PY
import json
d=json.load(open("gpurun_out/ab_${T}.json")); s=d["stages_ms_per_step"]
print("$L $e rep$rep", d["ms_per_step"], "grad", s["gradient"], "order", s["order"], "crit", s["critical"], "d0", s["d0"], "dtop", s["dtop"])
PY
  done
done
done
