mkdir -p gpurun_out
timeout 300 python scripts/time_stream.py 266 256 32 20 > gpurun_out/time266.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/st266.csv python scripts/prof_stream.py 266 256 32 2 > gpurun_out/st266.log 2>&1
cat gpurun_out/time266.log; python scripts/stream_summary.py gpurun_out/st266.csv 2>&1 | tail -n 12
