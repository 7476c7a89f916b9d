mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rows" -s 1 -c 1 -o gpurun_out/rows266b python scripts/prof_stream.py 266 256 32 2 > gpurun_out/rows_ncu.log 2>&1
tail -n 2 gpurun_out/rows_ncu.log
