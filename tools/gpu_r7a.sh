# last check of the tree: GPU suite, smoke, c4 bench, five-tetrahedra bench lines
T=${1:-r7a}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/${T}_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu.log
timeout 600 python bench.py > gpurun_out/bench_${T}_c4.json 2> gpurun_out/bench_${T}_c4.err
for cfg in c4 c3; do
  timeout 600 python bench.py --config $cfg --complex 5tet > gpurun_out/bench_${T}_${cfg}_5tet.json 2> gpurun_out/bench_${T}_${cfg}_5tet.err || echo "bench 5tet $cfg failed"
done
tail -n 3 gpurun_out/${T}_gpu.log
