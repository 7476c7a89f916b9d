mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/st100.csv python scripts/prof_stream.py 100 100 10 3 > gpurun_out/st100.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/st266.csv python scripts/prof_stream.py 266 256 32 2 > gpurun_out/st266.log 2>&1
tail -n 2 gpurun_out/st100.log gpurun_out/st266.log
