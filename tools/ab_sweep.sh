# A/B sweep of one environment knob (run under gpurun from the repo root): the GPU
# parity + full-size tests first, then bench.py per config and knob value.
# Usage: bash tools/ab_sweep.sh <VAR> "<values>" "<configs>"
#   e.g. bash tools/ab_sweep.sh DMS_ORDER_CTAS "0 1 2 4" "c4 c3"
# Prints: config VAR=value  M-vertices/s  ms/step  order-ms  gradient-ms  e2e-M-vertices/s
VAR=${1:?knob}
VALS=${2:?values}
CFGS=${3:-c4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t_par.log 2>&1
echo "parity=$?"
for cfg in $CFGS; do
  for v in $VALS; do
    echo "$cfg $VAR=$v $(env $VAR=$v timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); s=d["stages_ms_per_step"]; print(d["value"], d["ms_per_step"], s["order"], s.get("gradient"), d["e2e"]["value"])')"
  done
done
