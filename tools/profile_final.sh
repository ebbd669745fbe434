# Final round-2 capture (run under gpurun from the repo root): the GPU suite, bench lines for
# every config, ncu launch lists and --set full captures of the dominant kernels.
set -x
T=${1:-r2f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/${T}_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu.log
timeout 600 python bench.py > gpurun_out/bench_${T}_c4.json 2> gpurun_out/bench_${T}_c4.err
for cfg in c3 c5a c5b c2 c1; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${T}_$cfg.json 2> gpurun_out/bench_${T}_$cfg.err || echo "bench $cfg failed"
done
for cfg in c4 c3; do
  timeout 600 python bench.py --config $cfg --complex 5tet > gpurun_out/bench_${T}_${cfg}_5tet.json 2> gpurun_out/bench_${T}_${cfg}_5tet.err || echo "bench 5tet $cfg failed"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${T}_reference.json 2>&1
for cfg in c4 c3 c5a c5b; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$cfg.csv \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/ncu_l_$cfg.log 2>&1 || echo "launch list $cfg failed"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_pool -c 1 -o gpurun_out/${T}_k_gradient_pool3_c4 \
  python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/ncu_full_grad.log 2>&1 || echo "full grad failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_os_pass -s 1 -c 1 -o gpurun_out/${T}_k_os_pass_c4 \
  python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/ncu_full_os.log 2>&1 || echo "full os failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_uf_coop -c 1 -o gpurun_out/${T}_k_uf_coop_c5b \
  python bench.py --config c5b --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_uf.log 2>&1 || echo "full uf failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_d1_bigc -s 6 -c 1 -o gpurun_out/${T}_k_d1_bigc_c4_256 \
  python tools/d1_stats.py c4 256,256,256 > gpurun_out/ncu_full_d1.log 2>&1 || echo "full d1 failed"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_gradient|k_os_pass" --csv python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/${T}_ncu_grad_c4.csv 2>&1
ls -la gpurun_out
