# five-tetrahedra complex: GPU parity + the Freudenthal parity suites
T=${1:-r4b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_5tet.py -q -x --durations=8 > gpurun_out/${T}_t5.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_t5.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_rare_paths.py -q -x > gpurun_out/${T}_par.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_par.log
