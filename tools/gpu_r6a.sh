# full GPU suite on the current tree + bench lines (all configs, 5-tet on c3/c4)
T=${1:-r6a}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/${T}_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu.log
for cfg in c4 c3 c5a c5b c2 c1; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${T}_$cfg.json 2> gpurun_out/bench_${T}_$cfg.err || echo "bench $cfg failed"
done
for cfg in c4 c3; do
  timeout 600 python bench.py --config $cfg --complex 5tet > gpurun_out/bench_${T}_${cfg}_5tet.json 2> gpurun_out/bench_${T}_${cfg}_5tet.err || echo "bench 5tet $cfg failed"
done
tail -n 4 gpurun_out/${T}_gpu.log
