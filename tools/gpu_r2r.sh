mkdir -p gpurun_out
python tools/d1_stats.py c4 256,256,256 > gpurun_out/r2r_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_d1_bigc -s 6 -c 1 -o gpurun_out/r2r_bigc python tools/d1_stats.py c4 256,256,256 > gpurun_out/r2r_ncu.log 2>&1
