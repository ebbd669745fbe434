# ncu source-level capture of the five-tetrahedra gradient kernel on c3
T=${1:-t5p}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_t5 -c 1 -o gpurun_out/${T}_t5 \
  python bench.py --config c3 --complex 5tet --steps 1 --warmup 0 --no-e2e > gpurun_out/${T}_ncu.log 2>&1 || echo "ncu failed"
ncu -i gpurun_out/${T}_t5.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_t5_sass.csv 2> /dev/null
ls -la gpurun_out | grep ${T}
