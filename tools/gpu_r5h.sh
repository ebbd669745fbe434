# 1D shortcut: 1D parity (small, random sweep, rare paths), c5b full-size digests, bench c5b
T=${1:-r5h}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_rare_paths.py -q -x > gpurun_out/${T}_par.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_par.log
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py tests/test_gpu_fullsize.py -q -x -k "c5b or 1d" > gpurun_out/${T}_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_full.log
for cfg in c5b; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_${T}_$cfg.json 2> gpurun_out/bench_${T}_$cfg.err || echo "bench $cfg failed"
done
tail -n 3 gpurun_out/${T}_par.log gpurun_out/${T}_full.log
python - <<PY
import json
for c in ("c5b",):
    try:
        d=json.load(open("gpurun_out/bench_${T}_%s.json"%c)); print(c, d["value"], d["ms_per_step"], d["e2e"]["value"], d["stages_ms_per_step"])
    except Exception as e: print(c, "failed", e)
PY
