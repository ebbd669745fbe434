mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_d1.py -x -q > gpurun_out/r2q_d1.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_d1.log; timeout 900 python -m pytest tests/test_gpu_d1.py -x -q -k "crops or c2" >> gpurun_out/r2q_d1.log 2>&1
for a in "c4 128,128,128" "c3 96,96,96" "c4 256,256,256" "c3 128,128,128" "c4" "c3"; do
  timeout 300 python tools/d1_stats.py $a >> gpurun_out/r2q_stats.log 2>&1
done
