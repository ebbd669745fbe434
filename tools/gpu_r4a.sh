# Re-entry check of HEAD: GPU suite, smoke, bench lines of c4 / c5b / c3.
T=${1:-r4a}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/${T}_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu.log
for cfg in c4 c5b c3 c5a; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${T}_$cfg.json 2> gpurun_out/bench_${T}_$cfg.err || echo "bench $cfg failed"
done
