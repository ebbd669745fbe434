mkdir -p gpurun_out
for a in "c4 128,128,128" "c3 96,96,96" "c4 256,256,256" "c3 128,128,128" "c4"; do
  timeout 300 python tools/d1_stats.py $a >> gpurun_out/r2p_stats.log 2>&1
done
