# Round-2 re-entry check: the full GPU suite, smoke, and the default bench line.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2m_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_gpu.log
timeout 600 python bench.py > gpurun_out/r2m_bench_c4.json 2> gpurun_out/r2m_bench_c4.err
for cfg in c3 c5a c5b; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/r2m_bench_$cfg.json 2> gpurun_out/r2m_bench_$cfg.err
done
