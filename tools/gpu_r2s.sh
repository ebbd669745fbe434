mkdir -p gpurun_out
for a in "c4 256,256,256" "c4"; do
  timeout 300 python tools/d1_stats.py $a >> gpurun_out/r2s_stats.log 2>&1
done
