# Round profile capture (run under gpurun from the repo root): bench lines for every
# config, ncu launch lists, and one --set full capture of the dominant 3D kernel.
# Usage: bash tools/profile_round.sh <tag>
set -x
T=${1:-r1}
mkdir -p gpurun_out
for cfg in c4 c3 c5a c5b c2 c1; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${T}_$cfg.json 2> gpurun_out/bench_${T}_$cfg.err || echo "bench $cfg failed"
done
for cfg in c4 c3 c5a c5b; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$cfg.csv \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l_$cfg.log 2>&1 || echo "launch list $cfg failed"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_pool -c 1 -o gpurun_out/${T}_k_gradient_pool3_c4 \
  python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c4.log 2>&1 || echo "full c4 failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_uf_coop -c 1 -o gpurun_out/${T}_k_uf_coop_c5b \
  python bench.py --config c5b --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c5b.log 2>&1 || echo "full c5b failed"
ls -la gpurun_out
