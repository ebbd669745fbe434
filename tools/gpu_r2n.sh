set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_d1.py -x -q --durations=10 > gpurun_out/r2n_d1.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_d1.log
