mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/plane_launches.csv python scripts/plane_prof.py > gpurun_out/plane_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_plane -s 20 -c 1 -o gpurun_out/plane_full python scripts/plane_prof.py > gpurun_out/plane_ncu_full.log 2>&1
python scripts/launch_summary.py gpurun_out/plane_launches.csv 2>&1 | head -30
