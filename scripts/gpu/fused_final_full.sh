mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_code_fused.*bool.1" -s 7 -c 1 -o gpurun_out/fused_final -f python scripts/prof_fused.py > gpurun_out/fused_final.log 2>&1
tail -n 2 gpurun_out/fused_final.log
