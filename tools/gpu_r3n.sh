mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_d1.py -x -q > gpurun_out/r3n.log 2>&1; echo "rc=$?" >> gpurun_out/r3n.log
for a in "c4 256,256,256" "c4" "c3"; do
  timeout 300 python tools/d1_stats.py $a 2>&1 | grep "wall\|bigc" >> gpurun_out/r3n_stats.log
done
