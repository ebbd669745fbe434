# A/B of prebuilt libraries in abx/ on bench c4 (and c3): tools/gpu_ab.sh TAG lib1 lib2 ...
T=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
for L in "$@"; do
  for cfg in c4; do
    DMS_LIB=$PWD/abx/$L timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-d1 --no-e2e > gpurun_out/ab_${T}_${L}_${cfg}_$rep.json 2>/dev/null
    python - <<PY
import json
d=json.load(open("gpurun_out/ab_${T}_${L}_${cfg}_$rep.json")); s=d["stages_ms_per_step"]
print("$L $cfg rep$rep", d["ms_per_step"], "grad", s["gradient"], "order", s["order"], "d0", s["d0"], "dtop", s["dtop"])
PY
  done
done
done
