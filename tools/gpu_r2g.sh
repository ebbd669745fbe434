set -x
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 ) > gpurun_out/r2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pytest.log
timeout 600 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
