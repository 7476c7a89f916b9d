mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_code_fused.*bool.1" -s 8 -c 2 -o gpurun_out/fusedS3 -f python scripts/prof_fused.py > gpurun_out/fusedS3.log 2>&1
tail -n 2 gpurun_out/fusedS3.log
