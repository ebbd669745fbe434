set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t_par.log 2>&1; echo par=$?
for cfg in c4 c5b c5a c3; do
 for rb in 0 4 5 6; do
  echo "$cfg rb=$rb $(DMS_RANK_BUCKETS=$rb timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["stages_ms_per_step"]["order"], d["stages_ms_per_step"].get("gradient"), d["e2e"]["value"])')"
 done
done
