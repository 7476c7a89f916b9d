mkdir -p gpurun_out
OCSC_FUSED_PROBE_DEBUG=1 timeout 120 python scripts/fused_info.py > gpurun_out/finfo2.txt 2>&1; cat gpurun_out/finfo2.txt
