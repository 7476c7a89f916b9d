mkdir -p gpurun_out
timeout 300 python scripts/prof_invert.py 100 5100 f64 > gpurun_out/inv_time.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_hist_invert_reg" -s 2 -c 1 -o gpurun_out/inv python scripts/prof_invert.py 100 5100 f64 > gpurun_out/inv_ncu.log 2>&1
cat gpurun_out/inv_time.log; tail -n 2 gpurun_out/inv_ncu.log
