mkdir -p gpurun_out
for v in 0 32 128 512; do
  for a in "c3" "c4"; do
    DMS_D1_ADDS=$v timeout 300 python tools/d1_stats.py $a 2>&1 | grep "wall" | sed "s/^/adds=$v /" >> gpurun_out/r3o.log
  done
done
