# quick iteration: 3D parity (small + c3 full-size digests), bench c4 / c3, gradient warp-instruction count
T=${1:-r5c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_d1.py -q -x > gpurun_out/${T}_par.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_par.log
timeout 600 python -m pytest tests/test_gpu_fullsize_oracle.py -q -x -k "c3 or c5a" > gpurun_out/${T}_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_full.log
for cfg in c4 c3; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-d1 > gpurun_out/bench_${T}_$cfg.json 2> gpurun_out/bench_${T}_$cfg.err || echo "bench $cfg failed"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none -k regex:"k_gradient" -c 1 --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/${T}_ncu_grad_c4.csv 2>&1
tail -3 gpurun_out/${T}_par.log gpurun_out/${T}_full.log
python - <<PY
import json
for c in ("c4","c3"):
    try:
        d=json.load(open("gpurun_out/bench_${T}_%s.json"%c)); print(c, d["value"], d["ms_per_step"], d["e2e"]["value"], d["stages_ms_per_step"])
    except Exception as e: print(c, "failed", e)
PY
grep -E "k_gradient" gpurun_out/${T}_ncu_grad_c4.csv | cut -d, -f5,12- | head
