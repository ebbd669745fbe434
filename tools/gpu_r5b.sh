# ncu source-level capture of the 3D gradient kernel on c4 (per-line instruction counts)
T=${1:-r5b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_pool -c 1 -o gpurun_out/${T}_grad \
  python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-d1 > gpurun_out/${T}_ncu.log 2>&1 || echo "ncu failed"
ncu -i gpurun_out/${T}_grad.ncu-rep --page source --csv > gpurun_out/${T}_grad_source.csv 2> gpurun_out/${T}_src.err
ncu -i gpurun_out/${T}_grad.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_grad_sass.csv 2>> gpurun_out/${T}_src.err
ls -la gpurun_out
