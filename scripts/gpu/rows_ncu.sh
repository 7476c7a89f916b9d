mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rows|k_cols" -s 3 -c 3 -o gpurun_out/rows266 python scripts/prof_stream.py 266 256 32 2 > gpurun_out/rows_ncu.log 2>&1
tail -n 3 gpurun_out/rows_ncu.log
