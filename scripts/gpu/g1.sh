set -x
mkdir -p gpurun_out
timeout 120 python scripts/fused_info.py > gpurun_out/finfo.txt 2>&1; cat gpurun_out/finfo.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or config or cfg1 or headline" > gpurun_out/gt_fused.txt 2>&1; tail -5 gpurun_out/gt_fused.txt
timeout 300 python bench.py --no-secondary > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; cat gpurun_out/bench_c.json; tail -3 gpurun_out/bench_c.err
OCSC_FUSED_SIDE=0 timeout 300 python bench.py --no-secondary > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; cat gpurun_out/bench_s.json
